set -x
ncu -f --set full --clock-control none --import-source on -k 'regex:k_ilu_apply2' --launch-skip 3 --launch-count 2 -o /tmp/r02_ilu_eis2 python tools/run_solve.py --config C5 --maxit 6 > gpurun_out/ilu_ncu.log 2>&1
echo rc=$?
ncu -i /tmp/r02_ilu_eis2.ncu-rep --page raw --csv > gpurun_out/r02_c5_ilu_eis_ncu_full_raw.csv 2>/dev/null
python tools/ncu_traffic.py gpurun_out/r02_c5_ilu_eis_ncu_full_raw.csv
python -m pytest tests -m gpu -q > gpurun_out/r02_gputest_final.log 2>&1
tail -3 gpurun_out/r02_gputest_final.log
python __graft_entry__.py smoke 2>&1 | tail -2
