set -x
mkdir -p gpurun_out
(lscpu; free -g; nproc; nvidia-smi) > gpurun_out/r02_host.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -s -k "full_size" > gpurun_out/r02_pytest_fullsize.log 2>&1; echo "fullsize rc=$?"
timeout 1800 python tools/full_parity.py --configs c5 --slabs 16 --verbose --out gpurun_out/r02_full_parity_c5.jsonl > gpurun_out/r02_full_parity_c5.log 2>&1; echo "c5 rc=$?"
