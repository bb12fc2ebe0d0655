# round-2 session-4 closing batch on the final build: tests, race check, bench lines, ncu evidence, variants
set -u
O=gpurun_out/final_s4d
mkdir -p $O
run() { local out=$1; shift; echo "== $*" >> $O/log.txt; timeout "$@" >> $O/$out 2>> $O/log.txt; echo "rc=$?" >> $O/log.txt; }
run pytest_gpu.log 900 python -m pytest tests -m gpu -q
run race_check_debug.txt 900 python tools/race_check.py --lib tools/ab/libcommet_debug.so
run race_check_drop1.txt 900 python tools/race_check.py --lib tools/ab/libcommet_debug_drop1.so --expect-fail
run race_check_product.txt 900 python tools/race_check.py --lib paper_2510_00884_b200/libcommet.so --repeats 10
run bench_c5.json 900 python bench.py
run bench_c3.json 600 python bench.py --config c3 --steps 60 --warmup 5
run bench_c4.json 600 python bench.py --config c4 --steps 20 --warmup 3
run variants_c3.jsonl 900 python tools/variant_bench.py
run ncu.log 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e
run ncu.log 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fused_kernel -s 8 -c 16 --csv --log-file $O/traffic_c5.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e
run ncu.log 1500 ncu -f --set full --clock-control none --import-source on -k regex:fused_kernel -s 16 -c 1 -o /tmp/final_s4d python tools/ab_bench.py c5 paper_2510_00884_b200/libcommet.so
python tools/ncu_summary.py /tmp/final_s4d.ncu-rep > $O/ncu_c5_summary.txt 2>&1
python tools/ncu_stall_lines.py /tmp/final_s4d.ncu-rep > $O/ncu_c5_lines.txt 2>&1
cat $O/log.txt; tail -2 $O/pytest_gpu.log
