# round-2 session-5 closing check of the final build: GPU suite, smoke, default bench line
set -u
O=gpurun_out/r2s5f
mkdir -p $O
run() { local out=$1; shift; echo "== $*" >> $O/log.txt; timeout "$@" >> $O/$out 2>> $O/log.txt; echo "rc=$?" >> $O/log.txt; }
run pytest_gpu.log 1200 python -m pytest tests -m gpu -q
run smoke.log 300 python -c "import __graft_entry__ as g; g.smoke()"
run bench_c5.json 900 python bench.py
cat $O/log.txt; tail -2 $O/pytest_gpu.log; cat $O/smoke.log
