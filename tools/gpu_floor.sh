mkdir -p gpurun_out
./tools/micro_floor > gpurun_out/floor.txt 2>&1; cat gpurun_out/floor.txt
