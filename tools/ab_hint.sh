set -x
python tools/store_probe.py > gpurun_out/store_probe.json 2> gpurun_out/store_probe.err
for r in 1 2; do
for v in "" _nohint _na; do
  for c in 2 4; do
    echo "== $v c$c r$r"
    if [ -z "$v" ]; then python tools/sweep.py --config $c --shapes default --reps 50 | tail -1; else STENCIL_B200_LIB=paper_1308_1343_b200/libstencil_b200$v.so python tools/sweep.py --config $c --shapes default --reps 50 | tail -1; fi
  done
done
done > gpurun_out/ab_hint.log 2>&1
