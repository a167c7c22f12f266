# The oracle's FULL single-core run at the benchmarked C5 next to the GPU step (tools/config_sweep.py, no extrapolation;
# ~120 GB of host RAM, ~50 min).  The OpenMP timing row is a run of its own: ORACLE_OMP=1 python tools/oracle_run.py C5
# (two oracle processes do not fit the box's 196 GB).
avail=$(awk '/MemAvailable/ {print int($2/1048576)}' /proc/meminfo)
if [ "$avail" -lt 170 ]; then echo "not enough host RAM for the full C5 oracle run"; exit 0; fi
SWEEP_NO_OMP=1 timeout 3450 python tools/config_sweep.py C5 > gpurun_out/r02_config_c5.jsonl 2> gpurun_out/sweep_c5.err
echo sweep rc=$?
tail -c 600 gpurun_out/sweep_c5.err
