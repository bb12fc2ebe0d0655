mkdir -p gpurun_out
timeout 900 python tools/ab_bench.py c5 paper_2510_00884_b200/libcommet.so > gpurun_out/r02_ncu_c5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 16 -c 1 -o gpurun_out/r02_final_c5 python tools/ab_bench.py c5 paper_2510_00884_b200/libcommet.so > gpurun_out/r02_ncu_c5.log 2>&1
echo "ncu rc=$?"
