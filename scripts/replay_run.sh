#!/bin/bash
# On the GPU box: dump one cfg2 step's ID batches, replay them per engine,
# and profile chosen batches.  Usage: scripts/replay_run.sh "<engines>" "<prof batches>" <prof engine>
cd "$(dirname "$0")/.."
mkdir -p /tmp/idd gpurun_out && rm -f /tmp/idd/*
SBX_ID_DUMP=/tmp/idd python scripts/phase_timing.py --reps 1 > gpurun_out/dump.log 2>&1
timeout 300 scripts/id_bench --replay /tmp/idd $1 > gpurun_out/replay.txt 2>&1
for b in $2; do ID_BATCH=$b timeout 100 scripts/id_bench_prof --replay /tmp/idd $3 > gpurun_out/prof_b$b.txt 2>&1; done
