mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02_pytest_gpu_call39.log 2>&1; echo "pytest rc=$?"
timeout 900 python tools/race_check.py --lib tools/ab/libcommet_debug.so > gpurun_out/r02_race_check_debug_eb2.txt 2>&1; echo "race debug rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_c5_eb2.json 2> gpurun_out/r02_bench_c5_eb2.err; echo "bench rc=$?"
