#!/usr/bin/env bash
# End-of-round measurement batch on one B200 (run under gpurun from the repo root):
# bench lines c5 (default) / c3 / c4, the twist-cube Newton table, the material-point
# sweep, the ncu launch list of the default bench and one `ncu --set full` capture of
# the fused kernel on c3.  Everything lands in gpurun_out/final/.
set -u
O=gpurun_out/final
mkdir -p $O
run() { echo "== $*" >> $O/log.txt; timeout "$@" >> $O/log.txt 2>&1; echo "rc=$?" >> $O/log.txt; }
run 900 python bench.py > $O/bench_c5.json
run 600 python bench.py --config c3 --steps 20 --warmup 5 > $O/bench_c3.json
run 600 python bench.py --config c4 --steps 10 --warmup 3 > $O/bench_c4.json
for n in 16 32 64; do run 600 python tools/newton_bench.py --n $n >> $O/newton_twist.jsonl; done
if [ "${FINAL_N128:-1}" = 1 ]; then run 1200 python tools/newton_bench.py --n 128 >> $O/newton_twist.jsonl; fi
run 600 python tools/material_sweep.py > $O/material_sweep.jsonl
# launch list of the default bench command (cold-cache, serialised: shares, not absolutes)
run 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e
# the fused kernel, full set, 1 launch after 8 warm-up launches (c3, colour launches)
run 1200 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 8 -c 1 \
    -o $O/prof_c3 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu --no-e2e
tail -c 3000 $O/log.txt
