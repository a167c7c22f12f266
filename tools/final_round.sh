# Round-end measurement pass on one B200: the S10 and C5 bench lines, the reference arm (per-config records:
# tools/config_sweep.py; GPU suite: pytest tests -m gpu).
set -x
python bench.py --config S10 > gpurun_out/r02_bench_s10.json 2> gpurun_out/bench_s10.err
python bench.py > gpurun_out/r02_bench_c5.json 2> gpurun_out/bench_c5.err
python bench.py --impl reference > gpurun_out/r02_bench_c5_reference.json 2> gpurun_out/bench_ref.err
python tools/config_sweep.py C1 C2 C3 C4 > gpurun_out/r02_configs.jsonl 2> gpurun_out/sweep.err
