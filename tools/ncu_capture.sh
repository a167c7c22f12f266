set -x
python tools/run_solve.py --config C5 --maxit 30 > gpurun_out/final_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_final_c5_launches.csv python tools/run_solve.py --config C5 --maxit 30 > gpurun_out/final_ncu1.log 2>&1
echo rc=$?
ncu --set full --clock-control none --import-source on -k 'regex:k_op_node_sym|k_op_cell|k_vc_sym|k_ilu_apply2|k_dcgs_update|k_mdot2|k_dscale|k_p7|k_step34|k_prolong|k_csr_vec' --launch-skip 120 --launch-count 60 -o /tmp/r02_final_c5_full python tools/run_solve.py --config C5 --maxit 12 > gpurun_out/final_ncu2.log 2>&1
echo rc=$?
ncu -i /tmp/r02_final_c5_full.ncu-rep --page raw --csv > gpurun_out/r02_final_c5_ncu_full_raw.csv 2>/dev/null
ls -la gpurun_out/
