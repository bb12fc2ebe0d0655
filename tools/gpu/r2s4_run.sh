set -u
O=gpurun_out/r2s4
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/log.txt
AB_NET=gt timeout 300 python tools/ab_bench.py c3 paper_2510_00884_b200/libcommet.so > $O/gt_c3.txt 2>&1
AB_NET=gt timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 8 -c 1 -o $O/gt_c3 python tools/ab_bench.py c3 paper_2510_00884_b200/libcommet.so > $O/ncu_gt.log 2>&1; echo "ncu gt rc=$?" >> $O/log.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 8 -c 1 -o $O/icnn_c3 python tools/ab_bench.py c3 paper_2510_00884_b200/libcommet.so > $O/ncu_icnn.log 2>&1; echo "ncu icnn rc=$?" >> $O/log.txt
tail -3 $O/pytest_gpu.log; cat $O/gt_c3.txt; cat $O/log.txt
