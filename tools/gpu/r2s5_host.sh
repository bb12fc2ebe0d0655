# round-2 session-5: commet_assemble_host (library-side e2e copies): its tests, the GPU suite, bench lines
set -u
O=gpurun_out/r2s5h
mkdir -p $O
run() { local out=$1; shift; echo "== $*" >> $O/log.txt; timeout "$@" >> $O/$out 2>> $O/log.txt; echo "rc=$?" >> $O/log.txt; }
run pytest_host.log 600 python -m pytest tests/test_gpu_host.py -q
run pytest_gpu.log 1200 python -m pytest tests -m gpu -q
run smoke.log 300 python -c "import __graft_entry__ as g; g.smoke()"
run bench_c5.json 900 python bench.py
run bench_c3.json 600 python bench.py --config c3 --steps 60 --warmup 5
run bench_c4.json 600 python bench.py --config c4 --steps 20 --warmup 3
cat $O/log.txt; tail -3 $O/pytest_host.log; tail -2 $O/pytest_gpu.log; cat $O/smoke.log
