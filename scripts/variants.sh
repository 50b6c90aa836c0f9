# time solve-kernel variants: bash scripts/variants.sh v1 v2 ...  (build/libfpr_b200_<v>.so; "base" = default lib)
for v in "$@"; do
  if [ "$v" = base ]; then L=""; else L=paper_2203_09284_b200/csrc/build/libfpr_b200_$v.so; fi
  for c in 2 1; do for e in ec fused; do
    echo -n "$v cfg$c $e: "; FPR_B200_LIB=$L timeout -s KILL 120 python scripts/profile_solve.py $e $c 3 2>&1 | tail -1 | cut -c1-110
  done; done
done
