set -u
O=gpurun_out/r2s4
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu_rs.log 2>&1; echo "pytest rc=$?" >> $O/log_v.txt
timeout 900 python tools/race_check.py --lib tools/ab/libcommet_debug.so > $O/race_check_debug.txt 2>&1; echo "debug rc=$?" >> $O/log_v.txt
timeout 900 python tools/race_check.py --lib tools/ab/libcommet_debug_drop1.so --expect-fail > $O/race_check_drop1.txt 2>&1; echo "drop1 rc=$?" >> $O/log_v.txt
timeout 900 python tools/race_check.py --lib paper_2510_00884_b200/libcommet.so --repeats 10 > $O/race_check_product.txt 2>&1; echo "product rc=$?" >> $O/log_v.txt
L="tools/ab/libcommet_rs0.so tools/ab/libcommet_rs1b.so"
AB_NET=icnnw32x2 timeout 600 python tools/ab_bench.py c3 $L $L > $O/ab_rs_3pass.txt 2>&1
AB_NET=icnnw16x2 timeout 600 python tools/ab_bench.py c3 $L >> $O/ab_rs_3pass.txt 2>&1
tail -3 $O/pytest_gpu_rs.log; cat $O/log_v.txt $O/ab_rs_3pass.txt; tail -2 $O/race_check_*.txt
