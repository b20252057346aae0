# the final bench line + reference arm + launch list (outputs in gpurun_out/*_$TAG*)
mkdir -p gpurun_out
TAG=${TAG:-bfin}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi_$TAG.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log; tail -1 gpurun_out/smoke_$TAG.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu --skip-config1 --skip-config5 --skip-config4a > gpurun_out/ncu_bench_$TAG.log 2>&1
python tools/launch_table.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt 2>&1
echo done
