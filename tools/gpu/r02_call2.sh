set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu_call2.log 2>&1; echo "pytest rc=$?"
AB_STAGES=1 timeout 600 python tools/ab_bench.py c3 tools/ab/libcommet_base.so tools/ab/libcommet_stageprof.so > gpurun_out/r02_ab_stages_c3.txt 2>&1
AB_STAGES=1 timeout 600 python tools/ab_bench.py c4 tools/ab/libcommet_base.so tools/ab/libcommet_stageprof.so > gpurun_out/r02_ab_stages_c4.txt 2>&1
