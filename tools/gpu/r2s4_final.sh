# round-2 (session 4) measurement batch: bench lines, launch list, full ncu capture of the c5 kernel
set -u
O=gpurun_out/final_s4
mkdir -p $O
run() { local out=$1; shift; echo "== $*" >> $O/log.txt; timeout "$@" >> $O/$out 2>> $O/log.txt; echo "rc=$?" >> $O/log.txt; }
run bench_c5.json 900 python bench.py
run bench_c3.json 600 python bench.py --config c3 --steps 20 --warmup 5
run bench_c4.json 600 python bench.py --config c4 --steps 10 --warmup 3
run ncu.log 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e
run ncu.log 1500 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 16 -c 1 \
    -o /tmp/final_c5 python tools/ab_bench.py c5 paper_2510_00884_b200/libcommet.so
python tools/ncu_summary.py /tmp/final_c5.ncu-rep > $O/ncu_c5_summary.txt 2>&1
python tools/ncu_stall_lines.py /tmp/final_c5.ncu-rep > $O/ncu_c5_lines.txt 2>&1
tail -c 2000 $O/log.txt; cat $O/bench_c5.json
