set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu_call8.log 2>&1; echo "pytest rc=$?"
timeout 600 python tools/sanitize_cases.py > gpurun_out/r02_sanitize_plain.log 2>&1; echo "sanitize plain rc=$?"
timeout 600 python tools/ab_bench.py c3 paper_2510_00884_b200/libcommet.so > gpurun_out/r02_ncu_c3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 16 -c 1 -o gpurun_out/r02_full_c3 python tools/ab_bench.py c3 paper_2510_00884_b200/libcommet.so > gpurun_out/r02_ncu_c3.log 2>&1
echo done
