# Round evidence: bench line, ncu launch lists (bench, one step) and ncu --set full
# captures of the sweep (DMMA cfg2 64 RHS, GEMV cfg3 1 RHS), the quad TSQR
# and the DMMA GEMM.  Run under gpurun from the repo root; summaries go to
# profiles/ via scripts/summarize_ncu.py.
set -x
python bench.py > gpurun_out/r01_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_bench.csv python bench.py > gpurun_out/ncu_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r01_launches_step.csv python scripts/phase_timing.py --reps 3 --profile-last > gpurun_out/ncu_step.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:sweep_flow_kernel -s 3 -c 1 -o gpurun_out/r01_sweep_dmma python scripts/sweep_bench.py --cfg cfg2 --nrhs 64 --reps 1 > gpurun_out/ncu_sd.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:sweep_flow_kernel -s 3 -c 1 -o gpurun_out/r01_sweep_gemv python scripts/sweep_bench.py --cfg cfg3 --nrhs 1 --reps 1 > gpurun_out/ncu_sg.log 2>&1
ID_CASE="app leaves" ncu --set full --import-source on --clock-control none -k regex:tsqr_quad -c 1 -o gpurun_out/r01_tsqr_quad scripts/id_bench 1 > gpurun_out/ncu_tq.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 20 -c 1 -o gpurun_out/r01_gemm python scripts/phase_timing.py --reps 1 > gpurun_out/ncu_gm.log 2>&1
ls -la gpurun_out
