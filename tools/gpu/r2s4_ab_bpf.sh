set -u
O=gpurun_out/r2s4
mkdir -p $O
L="tools/ab/libcommet_ku2.so tools/ab/libcommet_bpf.so tools/ab/libcommet_pd4ku4.so"
timeout 1500 python tools/ab_bench.py c5 $L > $O/ab_bpf_c5.txt 2>&1
timeout 600 python tools/ab_bench.py c3 $L > $O/ab_bpf_c3.txt 2>&1
timeout 600 python tools/ab_bench.py c4 $L > $O/ab_bpf_c4.txt 2>&1
cat $O/ab_bpf_*.txt
