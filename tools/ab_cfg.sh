# A/B of one configuration's default launch between the product library and
# experimental variants (CFG=<config> [SHAPE=...] bash tools/ab_cfg.sh <variant>...),
# three interleaved rounds.
cfg=${CFG:-5}
shape=${SHAPE:-default}
reps=${REPS:-30}
for r in 1 2 3; do
  echo "== base r$r"; python tools/sweep.py --config $cfg --shapes "$shape" --reps $reps | tail -1
  for v in "$@"; do
    echo "== $v r$r"; STENCIL_B200_LIB=paper_1308_1343_b200/libstencil_b200_$v.so python tools/sweep.py --config $cfg --shapes "$shape" --reps $reps | tail -1
  done
done
