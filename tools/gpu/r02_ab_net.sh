# usage: bash tools/gpu/r02_ab_net.sh OUTNAME CONFIG NETS LIB...   (A/B of analytic-network builds)
out=$1; cfg=$2; nets=$3; shift 3
mkdir -p gpurun_out
for n in $(echo $nets | tr , ' '); do
  echo "== AB_NET=$n" >> gpurun_out/$out.txt
  AB_NET=$n timeout 900 python tools/ab_bench.py $cfg "$@" >> gpurun_out/$out.txt 2>&1
done
