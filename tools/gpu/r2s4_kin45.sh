set -u
O=gpurun_out/r2s4
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_kin45.log 2>&1; echo "pytest rc=$?" >> $O/pytest_kin45.log
timeout 900 python tools/variant_bench.py > $O/variants_kin45.jsonl 2>&1
L="tools/ab/libcommet_cur2.so paper_2510_00884_b200/libcommet.so"
AB_NET=gt timeout 600 python tools/ab_bench.py c3 $L $L > $O/ab_kin45_gt.txt 2>&1
AB_NET=cann timeout 600 python tools/ab_bench.py c3 $L > $O/ab_kin45_cann.txt 2>&1
timeout 600 python tools/ab_bench.py c3 $L > $O/ab_kin45_c3.txt 2>&1
tail -2 $O/pytest_kin45.log; cat $O/ab_kin45_*.txt
python -c "
import json
for l in open('$O/variants_kin45.jsonl'):
    try: d=json.loads(l)
    except Exception: continue
    print(f\"{d['model']:40s} {d['kernel_ms']:7.3f} ms\")"
