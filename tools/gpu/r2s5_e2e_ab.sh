# round-2 session-5: read-back streams / chunks of commet_assemble_host, c5 and c4 e2e A/B
set -u
O=gpurun_out/r2s5ab
mkdir -p $O
for sc in "2 8" "3 12" "4 16" "2 32"; do
  set -- $sc
  COMMET_HOST_COPY_STREAMS=$1 COMMET_HOST_CHUNKS=$2 timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu > $O/c5_s$1_c$2.json 2>> $O/log.txt
  python -c "import json;d=json.loads(open('$O/c5_s$1_c$2.json').read().strip().splitlines()[-1]);print('c5 streams=$1 chunks=$2', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2), '%.3e'%d['e2e']['value'])" >> $O/ab.txt
done
cat $O/ab.txt; tail -3 $O/log.txt
