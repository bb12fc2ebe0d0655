set -u
O=gpurun_out/final_s4b
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/log.txt
timeout 900 python tools/race_check.py --lib paper_2510_00884_b200/libcommet.so --repeats 10 > $O/race_check_product.txt 2>&1; echo "race product rc=$?" >> $O/log.txt
sed -i 's#gpurun_out/final_s4#gpurun_out/final_s4b#' tools/gpu/r2s4_final.sh
bash tools/gpu/r2s4_final.sh > /dev/null 2>&1
tail -3 $O/pytest_gpu.log; tail -1 $O/race_check_product.txt; cat $O/log.txt
