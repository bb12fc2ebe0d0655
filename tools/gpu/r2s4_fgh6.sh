set -u
O=gpurun_out/r2s4
mkdir -p $O
L="tools/ab/libcommet_cur2.so tools/ab/libcommet_fgh6.so tools/ab/libcommet_fgh8.so"
timeout 1500 python tools/ab_bench.py c5 $L > $O/ab_fgh6_c5.txt 2>&1
timeout 600 python tools/ab_bench.py c3 $L $L > $O/ab_fgh6_c3.txt 2>&1
cat $O/ab_fgh6_*.txt
