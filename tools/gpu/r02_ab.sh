# usage: bash tools/gpu/r02_ab.sh OUTNAME CONFIGS LIB...   (A/B of tools/ab builds)
out=$1; cfgs=$2; shift 2
mkdir -p gpurun_out
for c in $(echo $cfgs | tr , ' '); do
  timeout 900 python tools/ab_bench.py $c "$@" >> gpurun_out/$out.txt 2>&1
done
