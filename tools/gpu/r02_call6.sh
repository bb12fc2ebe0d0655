set -x
mkdir -p gpurun_out
timeout 900 python tools/ab_bench.py c3 tools/ab/libcommet_meta0.so tools/ab/libcommet_meta2.so tools/ab/libcommet_elem_meta0.so tools/ab/libcommet_elem_meta2.so tools/ab/libcommet_meta0.so tools/ab/libcommet_meta2.so > gpurun_out/r02_ab_meta2.txt 2>&1
timeout 900 python tools/ab_bench.py c4 tools/ab/libcommet_meta0.so tools/ab/libcommet_meta2.so tools/ab/libcommet_elem_meta0.so tools/ab/libcommet_elem_meta2.so >> gpurun_out/r02_ab_meta2.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu_call6.log 2>&1; echo "pytest rc=$?"
