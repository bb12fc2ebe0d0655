set -u
O=gpurun_out/r2s4
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_fgh.log 2>&1; echo "pytest rc=$?" >> $O/pytest_fgh.log
L="tools/ab/libcommet_cur2.so paper_2510_00884_b200/libcommet.so"
timeout 1500 python tools/ab_bench.py c5 $L > $O/ab_fgh_c5.txt 2>&1
timeout 600 python tools/ab_bench.py c3 $L $L > $O/ab_fgh_c3.txt 2>&1
timeout 600 python tools/ab_bench.py c4 $L > $O/ab_fgh_c4.txt 2>&1
tail -3 $O/pytest_fgh.log; cat $O/ab_fgh_*.txt
