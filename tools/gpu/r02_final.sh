mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02_final_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 900 python tools/race_check.py --lib tools/ab/libcommet_debug.so > gpurun_out/r02_final_race_check_debug.txt 2>&1; echo "race debug rc=$?"
timeout 900 python tools/race_check.py --lib paper_2510_00884_b200/libcommet.so --repeats 10 > gpurun_out/r02_final_race_check_product.txt 2>&1; echo "race product rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_final_bench_c5.json 2> gpurun_out/r02_final_bench_c5.err; echo "bench c5 rc=$?"
for c in c3 c4; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/r02_final_bench_$c.json 2> gpurun_out/r02_final_bench_$c.err; echo "bench $c rc=$?"
done
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/r02_final_ncu_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fused_kernel -s 8 -c 16 --csv --log-file gpurun_out/r02_final_launches_c5.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/r02_final_ncu.log 2>&1
echo "ncu rc=$?"
