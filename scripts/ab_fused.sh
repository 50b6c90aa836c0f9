# A/B of async (fused) solve variants on config 2 (and 3): bash scripts/ab_fused.sh v1 v2 ...
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = base ]; then L=""; else L=paper_2203_09284_b200/csrc/build/libfpr_b200_$v.so; fi
  for c in 2 3; do
  echo -n "$v cfg$c: "; FPR_B200_LIB=$L timeout -s KILL 120 python scripts/profile_solve.py fused $c 3 2>&1 | tail -1 | cut -c1-75
  done
done; done
