# Full round evidence on one GPU: smoke, GPU tests, ncu --set full of the
# sweep / stage / Pareto kernels (-> per-kernel DRAM traffic, used by the
# bench line's roofline), bench (+ CPU baseline), reference arm, launch
# list, phase probe, e2e probe.  Outputs in gpurun_out/*_$TAG*.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi_$TAG.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"g4_|bucket_min|suffix_min|pareto_select" -s 6 -c 8 -o gpurun_out/full_$TAG python tools/prof_sweep.py > gpurun_out/full_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_step -s 2 -c 2 -o gpurun_out/stage_$TAG python tools/prof_stage.py > gpurun_out/stage_$TAG.log 2>&1
python tools/traffic.py gpurun_out/traffic_$TAG.json gpurun_out/full_$TAG.ncu-rep gpurun_out/stage_$TAG.ncu-rep > /dev/null 2>&1 && cp gpurun_out/traffic_$TAG.json profiles/r1_traffic.json
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu --skip-config1 > gpurun_out/ncu_bench_$TAG.log 2>&1
timeout 300 python tools/phase_probe.py > gpurun_out/phase_$TAG.txt 2>&1
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_$TAG.txt 2>&1
timeout 300 python tools/launch_probe.py > gpurun_out/launch_probe_$TAG.txt 2>&1
echo done
