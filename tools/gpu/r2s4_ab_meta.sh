set -u
O=gpurun_out/r2s4
mkdir -p $O
L="tools/ab/libcommet_me0.so tools/ab/libcommet_me1.so tools/ab/libcommet_me2.so"
AB_NET=gt timeout 600 python tools/ab_bench.py c3 $L $L > $O/ab_meta_gt.txt 2>&1
AB_NET=cann timeout 600 python tools/ab_bench.py c3 $L > $O/ab_meta_cann.txt 2>&1
timeout 600 python tools/ab_bench.py c3 $L $L > $O/ab_meta_icnn.txt 2>&1
timeout 1200 python tools/ab_bench.py c5 tools/ab/libcommet_me0.so tools/ab/libcommet_me1.so > $O/ab_meta_c5.txt 2>&1
cat $O/ab_meta_*.txt
