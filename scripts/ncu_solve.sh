# ncu --set full capture of one persistent solve launch: bash scripts/ncu_solve.sh <engine> <config> <tag>
E=${1:-ec}; C=${2:-2}; T=${3:-r1}
timeout -s KILL 300 python scripts/profile_solve.py $E $C 1 > gpurun_out/plain_$T.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:solve_kernel -c 1 \
  -o gpurun_out/prof_$T python scripts/profile_solve.py $E $C 1 > gpurun_out/ncu_$T.log 2>&1
echo rc=$?; tail -3 gpurun_out/ncu_$T.log; cat gpurun_out/plain_$T.log | cut -c1-200
