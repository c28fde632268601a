mkdir -p gpurun_out
: > gpurun_out/exp43.log
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 >> gpurun_out/exp43.log
for v in r1d cur; do for c in c4 c1 c3; do
L=build_variants/libunigpu_$v.so; [ $v = cur ] && L=paper_2111_08692_b200/libunigpu.so
UG_LIB_OVERRIDE=$L OPS=utf16le_to_utf8 timeout -s KILL 120 python tools/opbench.py $c 1024 10 2>&1 | tail -1 >> gpurun_out/exp43.log
done; done
timeout -s KILL 600 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_case.py > gpurun_out/exp43_race.log 2>&1; echo "race rc=$?" >> gpurun_out/exp43.log
timeout -s KILL 600 compute-sanitizer --tool synccheck python tools/sanitize_case.py > gpurun_out/exp43_sync.log 2>&1; echo "sync rc=$?" >> gpurun_out/exp43.log
timeout -s KILL 600 compute-sanitizer --tool memcheck python tools/sanitize_case.py > gpurun_out/exp43_mem.log 2>&1; echo "mem rc=$?" >> gpurun_out/exp43.log
