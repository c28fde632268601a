cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest tests/test_gpu_planned.py tests/test_gpu_parity.py -x -q -k "planned or sharded_c_entry or binding or length_ex or same_stream or bounded" > gpurun_out/p1_pytest.log 2>&1; echo "pytest=$?"; tail -15 gpurun_out/p1_pytest.log
for c in c4:1024 c1:1024 c3:512 c2b:256; do OPS=utf8_to_utf16le,utf8_to_utf16le_planned,utf16le_to_utf8,utf16le_to_utf8_planned,plan8,plan16,utf16_length_from_utf8,utf8_length_from_utf16le timeout 300 python tools/opbench.py ${c%:*} ${c#*:} 20 2>&1 | tail -1; done > gpurun_out/p1_ops.log
cat gpurun_out/p1_ops.log
