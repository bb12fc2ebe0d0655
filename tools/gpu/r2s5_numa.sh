# round-2 session-5: e2e with the pinned host buffers on the GPU's NUMA node (two default c5 runs)
set -u
O=gpurun_out/r2s5n
mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1; lscpu | grep -i numa >> $O/topo.txt
for i in 1 2; do
  timeout 600 python bench.py > $O/bench_c5_$i.json 2>> $O/log.txt
  python -c "import json;d=json.loads(open('$O/bench_c5_$i.json').read().strip().splitlines()[-1]);e=d['e2e'];print('run $i', round(d['ms_per_step'],2), round(e['ms_per_step'],2), '%.3e'%e['value'], e.get('host_buffers_cpus'))" >> $O/ab.txt
done
cat $O/ab.txt $O/topo.txt; tail -3 $O/log.txt
