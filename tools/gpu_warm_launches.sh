# per-kernel durations with caches NOT flushed between kernels (warm, like the graph)
set -x
mkdir -p gpurun_out
TAG=${TAG:-warm}
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu --skip-stage > gpurun_out/ncu_$TAG.log 2>&1
echo done
