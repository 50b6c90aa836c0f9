set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -30
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout -s KILL 300 python bench.py --steps 20 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench_rc=$?
tail -5 gpurun_out/bench1.err; cat gpurun_out/bench1.json
