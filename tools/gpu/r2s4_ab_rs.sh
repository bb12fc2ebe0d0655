set -u
O=gpurun_out/r2s4
mkdir -p $O
L="tools/ab/libcommet_rs0.so tools/ab/libcommet_rs1.so"
timeout 600 python tools/ab_bench.py c3 $L $L > $O/ab_rs_c3.txt 2>&1
timeout 600 python tools/ab_bench.py c4 $L > $O/ab_rs_c4.txt 2>&1
timeout 1200 python tools/ab_bench.py c5 $L > $O/ab_rs_c5.txt 2>&1
cat $O/ab_rs_c3.txt $O/ab_rs_c4.txt $O/ab_rs_c5.txt
