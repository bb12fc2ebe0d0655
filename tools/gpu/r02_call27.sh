mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "saturated" > gpurun_out/r02_pytest_saturated.log 2>&1; echo "pytest rc=$?"
for c in c3 c4; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err; echo "bench $c rc=$?"
done
timeout 900 python bench.py --config c3 --jitter 0.1 --steps 20 --warmup 5 --no-cpu > gpurun_out/r02_bench_c3_jitter.json 2> gpurun_out/r02_bench_c3_jitter.err; echo "bench c3 jitter rc=$?"
