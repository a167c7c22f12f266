# Full oracle runs at the benchmarked C5 (no extrapolation), one after the other (each needs ~120 GB of host RAM):
# the OpenMP timing row first, then tools/config_sweep.py (GPU step + single-core oracle, parity fields).
free -g | head -2; nproc
avail=$(awk '/MemAvailable/ {print int($2/1048576)}' /proc/meminfo)
if [ "$avail" -lt 170 ]; then echo "not enough host RAM for the full C5 oracle run"; exit 0; fi
ORACLE_OMP=1 OMP_NUM_THREADS=$(nproc) timeout 3000 python tools/oracle_run.py C5 > gpurun_out/r02_oracle_omp_c5.json 2> gpurun_out/omp_c5.err
echo omp rc=$?; cat gpurun_out/r02_oracle_omp_c5.json
SWEEP_NO_OMP=1 timeout 5400 python tools/config_sweep.py C5 > gpurun_out/r02_config_c5.jsonl 2> gpurun_out/sweep_c5.err
echo sweep rc=$?
tail -c 600 gpurun_out/sweep_c5.err
