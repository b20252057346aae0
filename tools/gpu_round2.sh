# Round-2 final evidence on one GPU (outputs gpurun_out/*_$TAG*): smoke, the GPU
# suite, ncu --set full of the headline / stage / head kernels (-> DRAM traffic
# per launch for the bench's roofline), the bench line, the reference arm, the
# bench's launch list, the phase probe.
set -x
mkdir -p gpurun_out profiles/r2
TAG=${TAG:-r2f}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi_$TAG.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -q -m gpu --durations=20 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"g4_|pareto_select" -s 6 -c 8 -o gpurun_out/full_$TAG python tools/prof_sweep.py > gpurun_out/full_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_step -s 2 -c 2 -o gpurun_out/stage_$TAG python tools/prof_stage.py > gpurun_out/stage_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:head_certainty -s 3 -c 1 -o gpurun_out/head_$TAG python tools/head_probe.py > gpurun_out/headp_$TAG.log 2>&1
python tools/traffic.py profiles/r2/traffic.json gpurun_out/full_$TAG.ncu-rep gpurun_out/stage_$TAG.ncu-rep gpurun_out/head_$TAG.ncu-rep > gpurun_out/traffic_$TAG.log 2>&1
python tools/ncu_summary.py gpurun_out/full_$TAG.ncu-rep > gpurun_out/ncu_summary_$TAG.txt 2>&1
python tools/ncu_summary.py gpurun_out/stage_$TAG.ncu-rep >> gpurun_out/ncu_summary_$TAG.txt 2>&1
python tools/ncu_summary.py gpurun_out/head_$TAG.ncu-rep >> gpurun_out/ncu_summary_$TAG.txt 2>&1
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu --skip-config1 --skip-config5 --skip-config4a > gpurun_out/ncu_bench_$TAG.log 2>&1
python tools/launch_table.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt 2>&1
timeout 600 python tools/phase_probe.py > gpurun_out/phase_$TAG.txt 2>&1
echo done
