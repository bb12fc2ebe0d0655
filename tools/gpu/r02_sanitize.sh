# usage: bash tools/gpu/r02_sanitize.sh TOOL   (one compute-sanitizer tool per gpurun call)
tool=$1
mkdir -p gpurun_out
timeout 2400 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 200 python tools/sanitize_cases.py > gpurun_out/r02_sanitizer_$tool.txt 2>&1
echo "compute-sanitizer $tool rc=$?" | tee -a gpurun_out/r02_sanitizer_$tool.txt
