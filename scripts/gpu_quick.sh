# quick GPU cycle: parity tests, solve timings for configs 1-3, bench
timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for c in 1 2; do for e in ec fused lockstep; do timeout -s KILL 120 python scripts/profile_solve.py $e $c 3 2>&1 | tail -1; done; done
timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
