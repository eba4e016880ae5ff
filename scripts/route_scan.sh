# ID-engine routing scan on the batches of one real cfg2 step (diagnostic):
# dump every batch (SBX_ID_DUMP), then replay the auto routing under each
# setting of the crowded-TSQR knobs.
mkdir -p /tmp/iddump && rm -f /tmp/iddump/*
SBX_ID_DUMP=/tmp/iddump python scripts/phase_timing.py --reps 1 > /dev/null 2>&1
for v in "" "SBX_TSQR_MAXN=128" "SBX_TSQR_MAXN=128 SBX_TSQR_MAXSTEPS=800" "SBX_TSQR_MAXN=128 SBX_TSQR_MAXSTEPS=600" "SBX_TSQR_MAXN=128 SBX_TSQR_MAXSTEPS=400"; do
  echo "== $v"
  env $v scripts/id_bench --replay /tmp/iddump 0 | grep -v "^batch   [0-8] "
done
