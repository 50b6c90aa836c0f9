# Round profile artefacts for the bench command: plain run, ncu launch list, one full capture.
T=${1:-r1}
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-ingest --no-large"
timeout -s KILL 300 $CMD > gpurun_out/plain_bench_$T.json 2> gpurun_out/plain_bench_$T.err && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_$T.csv $CMD > gpurun_out/ncu_launch_$T.log 2>&1
echo launch_rc=$?
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:solve_kernel -c 1 \
   -o gpurun_out/bench_full_$T $CMD > gpurun_out/ncu_full_$T.log 2>&1
echo full_rc=$?
tail -2 gpurun_out/ncu_full_$T.log
# ingest leg (text -> CSR) launch list
(cd scripts && REPS=1 timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file ../gpurun_out/launches_ingest_$T.csv python ingest_once.py > ../gpurun_out/ncu_ingest_$T.log 2>&1)
echo ingest_rc=$?
