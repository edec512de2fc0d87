O=gpurun_out/evidence2
mkdir -p $O
python tools/profile_vcycle.py 256 3 > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_sweep_df -s 0 -c 1 -o $O/full_k_sweep_df_l0 python tools/profile_vcycle.py 256 3 > $O/log1 2>&1
ncu -i $O/full_k_sweep_df_l0.ncu-rep --page raw --csv > $O/raw_k_sweep_df_l0.csv 2>/dev/null
python tools/profile_solve.py C2 > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_cgs_sweep -s 20 -c 1 -o $O/full_k_cgs python tools/profile_solve.py C2 > $O/log2 2>&1
ncu -i $O/full_k_cgs.ncu-rep --page raw --csv > $O/raw_k_cgs.csv 2>/dev/null
ncu --set full --import-source on --clock-control none -k regex:k_block_inverse -c 1 -o $O/full_k_block_inverse python tools/profile_solve.py C2 > $O/log3 2>&1
ncu -i $O/full_k_block_inverse.ncu-rep --page raw --csv > $O/raw_k_block_inverse.csv 2>/dev/null
python tools/profile_solve.py C4 > $O/c4.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:"k_plain_tiles|k_big_phase|k_residual_restrict|k_cgs_sweep" -s 40 -c 6 -o $O/full_c4 python tools/profile_solve.py C4 > $O/log4 2>&1
ncu -i $O/full_c4.ncu-rep --page raw --csv > $O/raw_c4.csv 2>/dev/null
ls $O
