mkdir -p gpurun_out
bash tools/quick.sh q5 > gpurun_out/exp15.log 2>&1
bash tools/prof3.sh val8 utf8_validate k_validate >> gpurun_out/exp15.log 2>&1
