mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/exp41_t.log
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 > gpurun_out/exp41_bench.json 2> gpurun_out/exp41_bench.err
