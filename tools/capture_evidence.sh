#!/bin/bash
# Round evidence (current code) on one B200 through gpurun: bench lines (C2 headline with
# cpu_baseline, reference arm, C3/C4/C5, slab-partitioned C3/C4 with the slabs sharing the
# GPU), the ncu launch list of the C2 bench command, DRAM bytes per launch of each config's
# roofline kernels, and --set full captures of the C2 dataflow sweep and the C4 fine-level
# band-major plain phase.  Each ncu pass runs only after the same command exited 0 without
# ncu.  Output: gpurun_out/ev4/
set -u
O=gpurun_out/ev4
mkdir -p $O
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err || exit 1
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
python bench.py --config C3 --slabs 4 --steps 5 --warmup 3 > $O/bench_c3_slabs4.json 2> $O/bench_c3_slabs4.err
python bench.py --config C4 --slabs 2 --steps 2 --warmup 3 > $O/bench_c4_slabs2.json 2> $O/bench_c4_slabs2.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/c2_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
python tools/profile_solve.py C4 > /dev/null 2>&1 || exit 1
ncu --metrics $M --clock-control none -k regex:"k_plain_df|k_big_phase|k_ortho|k_residual_restrict|k_stokes_apply|k_prolong_add|k_scale_by_norm" \
    -c 90 --csv --log-file $O/c4_traffic.csv python tools/profile_solve.py C4 > $O/ncu_c4.log 2>&1
python tools/profile_vcycle.py 256 3 > /dev/null 2>&1 || exit 1
ncu --metrics $M --clock-control none -k regex:k_sweep_df -c 6 --csv --log-file $O/c2_sweep_df.csv \
    python tools/profile_vcycle.py 256 3 > /dev/null 2>&1
python tools/profile_solve.py C3 > /dev/null 2>&1 || exit 1
ncu --metrics $M --clock-control none -k regex:"k_sweep_df|k_plain_df|k_big_phase" -c 24 --csv \
    --log-file $O/c3_traffic.csv python tools/profile_solve.py C3 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_sweep_df -s 0 -c 1 -o $O/full_k_sweep_df \
    python tools/profile_vcycle.py 256 3 > $O/ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_plain_df -s 0 -c 1 -o $O/full_k_plain_df \
    python tools/profile_solve.py C4 > $O/ncu_full2.log 2>&1
ncu -i $O/full_k_sweep_df.ncu-rep --page details --csv > $O/full_k_sweep_df_details.csv 2>/dev/null
ncu -i $O/full_k_plain_df.ncu-rep --page details --csv > $O/full_k_plain_df_details.csv 2>/dev/null
ls -la $O
