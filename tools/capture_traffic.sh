#!/bin/bash
# DRAM bytes per launch of the roofline kernels (ncu --set full is not needed:
# two dram counters), for profiles/traffic.json.  Output: gpurun_out/traffic/
O=gpurun_out/traffic
mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
python tools/profile_vcycle.py 256 3 > /dev/null 2>&1 || exit 1
ncu --metrics $M --clock-control none -k regex:k_sweep_df -c 6 --csv --log-file $O/c2_sweep_df.csv python tools/profile_vcycle.py 256 3 > /dev/null 2>&1
python tools/profile_solve.py C4 > /dev/null 2>&1 || exit 1
ncu --metrics $M --clock-control none -k regex:"k_plain_tiles|k_big_phase" -c 24 --csv --log-file $O/c4_tiles.csv python tools/profile_solve.py C4 > /dev/null 2>&1
python tools/profile_step.py C3 > /dev/null 2>&1 || exit 1
ncu --metrics $M --clock-control none -k regex:"k_sweep_df|k_plain_tiles|k_big_phase" -c 24 --csv --log-file $O/c3.csv python tools/profile_solve.py C3 > /dev/null 2>&1
ls -la $O
