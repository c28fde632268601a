cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG:-r2a}_pytest.log 2>&1; echo "pytest=$?"
tail -5 gpurun_out/${TAG:-r2a}_pytest.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG:-r2a}_smoke.log 2>&1; echo "smoke=$?"
