mkdir -p gpurun_out
cp paper_2111_08692_b200/libunigpu.so gpurun_out/lib_cf1.so
OPS=utf16le_to_utf8 timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:k_transcode16 -s 1 -c 1 -o gpurun_out/cf1 python tools/opbench.py c1 1024 2 > gpurun_out/exp38.log 2>&1
echo "rc=$?" >> gpurun_out/exp38.log
