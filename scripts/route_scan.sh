# ID-engine routing scan on the batches of one real cfg2 step (diagnostic):
# dump every batch (SBX_ID_DUMP), then replay it under the auto routing and
# each forced engine (scripts/id_bench.cu --replay).
mkdir -p /tmp/iddump && rm -f /tmp/iddump/*
SBX_ID_DUMP=/tmp/iddump python scripts/phase_timing.py --reps 1 > /dev/null 2>&1
scripts/id_bench --replay /tmp/iddump ${ENGINES:-0 1 2 3 4 5 6} | grep -v "^batch   [0-8] "
