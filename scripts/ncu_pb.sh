#!/bin/bash
# ncu metrics of the propagation-blocked sweep kernels: scripts/ncu_pb.sh <config> <out.csv>
ncu --clock-control none -k regex:"pb_(gather|accum)" -c 2 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_requests.sum,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__cycles_active.avg,sm__cycles_elapsed.max,smsp__cycles_active.max --csv python scripts/pb_once.py "$1" > "$2" 2>&1
