# Round-end measurement pass on one B200: per-config records, the S10 and C5 bench lines, the reference arm, the GPU suite.
set -x
python tools/config_sweep.py C1 C2 C3 C4 > gpurun_out/r02_configs.jsonl 2> gpurun_out/sweep.err
python bench.py --config S10 > gpurun_out/r02_bench_s10.json 2> gpurun_out/bench_s10.err
python bench.py > gpurun_out/r02_bench_c5.json 2> gpurun_out/bench_c5.err
python bench.py --impl reference > gpurun_out/r02_bench_c5_reference.json 2> gpurun_out/bench_ref.err
python -m pytest tests -m gpu -q > gpurun_out/r02_gputest_final.log 2>&1
tail -3 gpurun_out/r02_gputest_final.log
python __graft_entry__.py smoke 2>&1 | tail -2
