for v in "" "SBX_SWEEP_NO_DIRECT=1" "SBX_GJ_DMMA128=0" "SBX_NO_THIN_GEMM=1" "SBX_GJ_SMEM=1" "SBX_NO_MALLOPT=1"; do
  echo "== $v"; env $v python bench.py --config cfg4 --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['ms_per_step'], d['details'].get('max_rel_velocity_error'), d['details'].get('max_k'))
"
done
