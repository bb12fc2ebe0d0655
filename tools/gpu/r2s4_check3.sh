set -u
O=gpurun_out/s4c
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/log.txt
timeout 900 python bench.py > $O/bench_c5.json 2>> $O/log.txt; echo "bench rc=$?" >> $O/log.txt
timeout 1500 ncu -f --set full --clock-control none --import-source on -k regex:fused_kernel -s 16 -c 1 -o /tmp/c5_s4c python tools/ab_bench.py c5 paper_2510_00884_b200/libcommet.so > $O/ncu_full.log 2>&1; echo "ncu rc=$?" >> $O/log.txt
python tools/ncu_summary.py /tmp/c5_s4c.ncu-rep > $O/ncu_c5_summary.txt 2>&1
python tools/ncu_stall_lines.py /tmp/c5_s4c.ncu-rep _ZN6commet12fused_kernelINS_3CfgILi64ELi16ELi8ELi8ELi3ELi0ELi0ELi0ELi4ELi0EEEEEvNS_7AsmArgsE 40 > $O/ncu_c5_lines.txt 2>&1
tail -2 $O/pytest_gpu.log; cat $O/log.txt
python -c "import json;d=json.loads(open('$O/bench_c5.json').read().strip().splitlines()[-1]);print(d['value'],d['kernel_ms_per_step'],d['roofline']['frac'],d['clocks'])"
