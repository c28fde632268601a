mkdir -p gpurun_out
timeout -s KILL 1300 python -m pytest tests -q -m gpu -x 2>&1 | tail -2 > gpurun_out/exp91.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 >> gpurun_out/exp91.log
bash tools/gpu_full.sh r1m
bash tools/allcfg.sh r1m
