set -u
O=gpurun_out/r2s4
mkdir -p $O
GTK=_ZN6commet12fused_kernelINS_3CfgILi16ELi32ELi8ELi8ELi3ELi1ELi1ELi0ELi4ELi0EEEEEvNS_7AsmArgsE
AB_NET=gt timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 8 -c 1 -o /tmp/gt_c3 python tools/ab_bench.py c3 paper_2510_00884_b200/libcommet.so > $O/ncu_gt.log 2>&1; echo "ncu gt rc=$?" >> $O/log.txt
python tools/ncu_summary.py /tmp/gt_c3.ncu-rep > $O/ncu_gt_summary.txt 2>&1
python tools/ncu_stall_lines.py /tmp/gt_c3.ncu-rep $GTK 40 > $O/ncu_gt_lines.txt 2>&1
ncu -i /tmp/gt_c3.ncu-rep --page raw --csv > $O/ncu_gt_raw.csv 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 8 -c 1 -o /tmp/icnn_c3 python tools/ab_bench.py c3 paper_2510_00884_b200/libcommet.so > $O/ncu_icnn.log 2>&1; echo "ncu icnn rc=$?" >> $O/log.txt
python tools/ncu_summary.py /tmp/icnn_c3.ncu-rep > $O/ncu_icnn_summary.txt 2>&1
python tools/ncu_stall_lines.py /tmp/icnn_c3.ncu-rep > $O/ncu_icnn_lines.txt 2>&1
ncu -i /tmp/icnn_c3.ncu-rep --page raw --csv > $O/ncu_icnn_raw.csv 2>&1
cat $O/log.txt; head -30 $O/ncu_gt_summary.txt
