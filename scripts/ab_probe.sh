# A/B of solve variants on config 2, interleaved: bash scripts/ab_probe.sh v1 v2 ... (base = default lib)
for rep in 1 2 3; do
for v in "$@"; do
  if [ "$v" = base ]; then L=""; else L=paper_2203_09284_b200/csrc/build/libfpr_b200_$v.so; fi
  echo -n "$v: "; FPR_B200_LIB=$L timeout -s KILL 120 python scripts/profile_solve.py ec 2 5 2>&1 | tail -1 | cut -c1-60
done; done
