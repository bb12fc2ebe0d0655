set -u
O=gpurun_out/r2s4
mkdir -p $O
COMMET_LIB=$PWD/tools/ab/libcommet_sig1.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "activation or parity_small" > $O/sig1_tests.log 2>&1; echo "sig1 tests rc=$?" >> $O/sig1_tests.log
L="tools/ab/libcommet_cur.so tools/ab/libcommet_sig1.so"
timeout 1500 python tools/ab_bench.py c5 $L > $O/ab_sig_c5.txt 2>&1
timeout 600 python tools/ab_bench.py c3 $L $L > $O/ab_sig_c3.txt 2>&1
timeout 600 python tools/ab_bench.py c4 $L > $O/ab_sig_c4.txt 2>&1
tail -3 $O/sig1_tests.log; cat $O/ab_sig_*.txt
