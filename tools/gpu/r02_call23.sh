set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu_call23.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_c5.json 2> gpurun_out/r02_bench_c5.err; echo "bench rc=$?"
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/r02_ncu_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fused_kernel -s 8 -c 16 --csv --log-file gpurun_out/r02_launches_c5.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/r02_ncu_launches.log 2>&1
echo done
