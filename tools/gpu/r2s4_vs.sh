set -u
O=gpurun_out/r2s4
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_material.py -q -x > $O/pytest_vs2.log 2>&1; echo "pytest rc=$?" >> $O/pytest_vs2.log
L="tools/ab/libcommet_cur4.so paper_2510_00884_b200/libcommet.so"
timeout 1500 python tools/ab_bench.py c5 $L > $O/ab_vs2_c5.txt 2>&1
timeout 600 python tools/ab_bench.py c3 $L $L > $O/ab_vs2_c3.txt 2>&1
timeout 600 python tools/ab_bench.py c4 $L > $O/ab_vs2_c4.txt 2>&1
tail -2 $O/pytest_vs2.log; cat $O/ab_vs2_*.txt
