# Round-2 profile refresh (one GPU call; outputs in gpurun_out/):
# smoke, the ncu launch list of the driver's bench command, and one
# `ncu --set full` capture per product kernel (C2 d4_all, C3 pairs LA + LB,
# C4 level Laplacian, C5 rhs24) at the default launch shapes.  Summaries:
#   python tools/ncu_summary.py gpurun_out/r02_*.ncu-rep > profiles/r02/ncu_kernels.json
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?" >> gpurun_out/smoke.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py --steps 20 --warmup 5 --no-cpu --sustained-steps 0 --e2e-steps 3 > gpurun_out/r02_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:d4_kernel -s 5 -c 1 -o gpurun_out/r02_c2_d4_all \
    python tools/sweep.py --config 2 --shapes 32,4,4,2 --reps 3 > gpurun_out/r02_ncu_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:rkpair_kernel -s 6 -c 2 -o gpurun_out/r02_c3_pairs \
    python tools/sweep.py --config 3 --shapes 32,4,64,1 --reps 3 > gpurun_out/r02_ncu_c3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:d4_kernel -s 5 -c 1 -o gpurun_out/r02_c4_level \
    python tools/sweep.py --config 4 --shapes 32,4,128,2 --reps 3 > gpurun_out/r02_ncu_c4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:rhs24_kernel -s 3 -c 1 -o gpurun_out/r02_c5_rhs24 \
    python tools/sweep.py --config 5 --shapes 32,24,192,1 --reps 2 > gpurun_out/r02_ncu_c5.log 2>&1
ls -la gpurun_out/
