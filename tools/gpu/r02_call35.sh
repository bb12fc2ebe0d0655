mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02_pytest_gpu_call35.log 2>&1; echo "pytest rc=$?"
timeout 900 python tools/variant_bench.py > gpurun_out/r02_variants_c3.jsonl 2>&1; echo "variants rc=$?"
