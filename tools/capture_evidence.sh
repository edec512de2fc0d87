#!/bin/bash
# Round-2 evidence on one B200 through gpurun (outputs in gpurun_out/ev3/):
# bench lines (C3 headline with cpu_baseline and the C4 secondary, reference
# arm, C2, C4, C5), the ncu launch list of the C3 bench command, DRAM bytes per
# launch of one C3 solve's kernels, --set full captures of the C3 dataflow
# sweep, the C4 band-major plain phase, the C4 fused apply (with structures) and
# the paper mode's lexicographic box sweep, the C4 operator probe and the paper
# mode's Table 2 through the C ABI.  Each ncu pass runs only after the same
# command exited 0 without ncu.
set -u
O=gpurun_out/ev3
mkdir -p $O
python bench.py > $O/bench_c3.json 2> $O/bench_c3.err || exit 1
python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
python bench.py --config C2 --steps 30 --warmup 3 --no-cpu-baseline --no-secondary > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
python bench.py --config C5 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
python tools/c4_ops_probe.py C4 > $O/c4_ops_probe.txt 2>&1
python tools/paper_mode_probe.py 64 > $O/paper_mode_table2.txt 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary"
$B > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 9000 --csv --log-file $O/c3_launches.csv $B > $O/ncu_launches.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
python tools/profile_solve.py C3 > /dev/null 2>&1 || exit 1
ncu --metrics $M --clock-control none -k regex:"k_sweep_df|k_plain_df|k_big_phase|k_coarse_cycle|k_residual_restrict|k_ortho|k_stokes_apply|k_prolong_add|k_canon_inverse" \
    -c 400 --csv --log-file $O/c3_traffic.csv python tools/profile_solve.py C3 > $O/ncu_c3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_sweep_df -s 0 -c 1 -o $O/full_k_sweep_df_c3 \
    python tools/profile_solve.py C3 > $O/ncu_full1.log 2>&1
python tools/profile_solve.py C4 > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_plain_df -s 0 -c 1 -o $O/full_k_plain_df_c4 \
    python tools/profile_solve.py C4 > $O/ncu_full2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_stokes_apply_t -s 2 -c 1 -o $O/full_k_stokes_apply_t_c4 \
    python tools/profile_solve.py C4 > $O/ncu_full3.log 2>&1
ncu --metrics $M --clock-control none -k regex:"k_plain_df|k_big_phase|k_residual_restrict_t|k_ortho|k_stokes_apply|k_prolong_add" \
    -c 120 --csv --log-file $O/c4_traffic.csv python tools/profile_solve.py C4 > $O/ncu_c4.log 2>&1
python tools/paper_mode_probe.py 64 > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_sweep -s 40 -c 1 -o $O/full_pm_k_sweep \
    python tools/paper_mode_probe.py 64 > $O/ncu_full4.log 2>&1
for f in full_k_sweep_df_c3 full_k_plain_df_c4 full_k_stokes_apply_t_c4 full_pm_k_sweep; do
  ncu -i $O/$f.ncu-rep --page details --csv > $O/${f}_details.csv 2>/dev/null
done
rm -f $O/*.ncu-rep
ls -la $O
