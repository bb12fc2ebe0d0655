set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu_call19.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench_c5_ws.json 2> gpurun_out/r02_bench_c5_ws.err; echo "bench rc=$?"
