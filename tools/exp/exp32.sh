mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -q -m gpu -x -k "host_pipeline" 2>&1 | tail -5 > gpurun_out/exp32_t1.log
timeout -s KILL 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/exp32_t2.log
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 > gpurun_out/exp32_bench.json 2> gpurun_out/exp32_bench.err
