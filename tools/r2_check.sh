cd $GRAFT_REPO_ROOT
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_pytest.log 2>&1; echo "pytest=$?"; tail -3 gpurun_out/r2b_pytest.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1; echo "smoke=$?"; tail -1 gpurun_out/r2b_smoke.log
timeout -s KILL 900 python bench.py --size-mib 2048 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench_small.log 2>&1; echo "bench=$?"; tail -c 3000 gpurun_out/r2b_bench_small.log
