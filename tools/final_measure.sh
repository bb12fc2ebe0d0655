#!/usr/bin/env bash
# End-of-round measurement batch on one B200 (run under gpurun from the repo root):
# bench lines c5 (default) / c3 / c4, the twist-cube Newton table, the material-point
# sweep, the ncu launch list of the default bench and one `ncu --set full` capture of
# the fused kernel on c3.  Everything lands in gpurun_out/final/.
set -u
O=gpurun_out/final
mkdir -p $O
# run OUT SECONDS CMD...: stdout appended to $O/OUT, stderr and the exit code to $O/log.txt
run() { local out=$1; shift; echo "== $*" >> $O/log.txt; timeout "$@" >> $O/$out 2>> $O/log.txt; echo "rc=$?" >> $O/log.txt; }
run bench_c5.json 900 python bench.py
run bench_c3.json 600 python bench.py --config c3 --steps 20 --warmup 5
run bench_c4.json 600 python bench.py --config c4 --steps 10 --warmup 3
for n in 16 32 64; do run newton_twist.jsonl 600 python tools/newton_bench.py --n $n; done
if [ "${FINAL_N128:-1}" = 1 ]; then run newton_twist.jsonl 1200 python tools/newton_bench.py --n 128; fi
run material_sweep.jsonl 600 python tools/material_sweep.py
# launch list of the default bench command (cold-cache, serialised: shares, not absolutes)
run ncu.log 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e
# the fused kernel, full set, 1 launch after 8 warm-up launches (c3, colour launches)
run ncu.log 1200 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 8 -c 1 \
    -o $O/prof_c3 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu --no-e2e
tail -c 3000 $O/log.txt
