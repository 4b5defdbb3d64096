# One GPU call: GPU tests, smoke, the default bench line, the reference arm,
# the ncu launch list of a short bench run and one full ncu capture of the
# headline kernel (d4_all, config 2 default launch).  Outputs in gpurun_out/.
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests=$?" >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
python bench.py --impl reference > gpurun_out/bench_ref.jsonl 2>> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 20 --warmup 3 --tune 10 --no-cpu --sustained-steps 0 --e2e-steps 3 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:d4_kernel -s 5 -c 1 -o gpurun_out/d4_full \
    python tools/sweep.py --config 2 --shapes 32,4,4,2 --reps 3 > gpurun_out/ncu_d4.log 2>&1
