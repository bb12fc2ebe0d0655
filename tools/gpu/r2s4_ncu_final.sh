set -u
O=gpurun_out/final_s4b
mkdir -p $O
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fused_kernel -s 8 -c 16 --csv --log-file $O/traffic_c5.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > $O/ncu_traffic.log 2>&1; echo "traffic rc=$?" >> $O/log2.txt
timeout 1500 ncu -f --set full --clock-control none --import-source on -k regex:fused_kernel -s 16 -c 1 -o /tmp/final_c5b python tools/ab_bench.py c5 paper_2510_00884_b200/libcommet.so > $O/ncu_full.log 2>&1; echo "full rc=$?" >> $O/log2.txt
python tools/ncu_summary.py /tmp/final_c5b.ncu-rep > $O/ncu_c5_summary.txt 2>&1
python tools/ncu_stall_lines.py /tmp/final_c5b.ncu-rep > $O/ncu_c5_lines.txt 2>&1
cat $O/log2.txt; head -24 $O/ncu_c5_summary.txt
