set -u
O=gpurun_out/r2s4
mkdir -p $O
L="tools/ab/libcommet_bpf.so tools/ab/libcommet_e8u2.so tools/ab/libcommet_t7r.so"
timeout 1500 python tools/ab_bench.py c5 $L > $O/ab_e8_c5.txt 2>&1
timeout 600 python tools/ab_bench.py c3 $L $L > $O/ab_e8_c3.txt 2>&1
AB_NET=gt timeout 600 python tools/ab_bench.py c3 $L > $O/ab_e8_gt.txt 2>&1
AB_NET=cann timeout 600 python tools/ab_bench.py c3 $L > $O/ab_e8_cann.txt 2>&1
cat $O/ab_e8_*.txt
