set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu_call4.log 2>&1; echo "pytest rc=$?"
timeout 900 python tools/ab_bench.py c3 tools/ab/libcommet_act6.so tools/ab/libcommet_act8.so tools/ab/libcommet_act6.so tools/ab/libcommet_act8.so > gpurun_out/r02_ab_act.txt 2>&1
timeout 900 python tools/ab_bench.py c4 tools/ab/libcommet_act6.so tools/ab/libcommet_act8.so >> gpurun_out/r02_ab_act.txt 2>&1
timeout 600 python tools/ab_bench.py c3 tools/ab/libcommet_elemonly.so > gpurun_out/r02_elemonly_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 16 -c 1 -o gpurun_out/r02_elemonly_c3 python tools/ab_bench.py c3 tools/ab/libcommet_elemonly.so > gpurun_out/r02_elemonly_ncu.log 2>&1
echo done
