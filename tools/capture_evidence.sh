#!/bin/bash
# Round evidence on one B200 (run through gpurun): bench lines, the reference
# arm, the ncu launch list of the C2 bench command and --set full captures of
# the top kernels.  Each ncu pass runs only after its command exited 0 without
# ncu.  Output: gpurun_out/evidence/
set -u
O=gpurun_out/evidence
mkdir -p $O
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err || exit 1
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
python bench.py --config C3 --steps 5 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/c2_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
python tools/profile_vcycle.py 256 3 > /dev/null 2>&1 || exit 1
for K in k_sweep_df k_coarse_cycle k_residual_restrict k_cgs_sweep k_block_inverse; do
  ncu --set full --import-source on --clock-control none -k regex:$K -s 2 -c 1 -o $O/full_$K \
      python tools/profile_vcycle.py 256 3 > $O/ncu_full_$K.log 2>&1
  ncu -i $O/full_$K.ncu-rep --page details --csv > $O/full_$K.csv 2>/dev/null
done
ls -la $O
