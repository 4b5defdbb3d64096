# A/B of C3 (RK4 Laplacian pairs, default shape) between the product library
# and experimental variants (args: variant suffixes), interleaved rounds.
shape=${SHAPE:-32,4,64,1}
for r in 1 2 3; do
  echo "== base r$r"; python tools/sweep.py --config 3 --shapes "$shape" --reps 100 | tail -1
  for v in "$@"; do
    echo "== $v r$r"; STENCIL_B200_LIB=paper_1308_1343_b200/libstencil_b200_$v.so python tools/sweep.py --config 3 --shapes "$shape" --reps 100 | tail -1
  done
done
