mkdir -p gpurun_out
timeout 900 python tools/race_check.py --lib tools/ab/libcommet_debug.so > gpurun_out/r02_race_check_debug.txt 2>&1; echo "debug rc=$?" | tee -a gpurun_out/r02_race_check_debug.txt
timeout 900 python tools/race_check.py --lib tools/ab/libcommet_debug_drop1.so --expect-fail > gpurun_out/r02_race_check_drop1.txt 2>&1; echo "drop1 rc=$?" | tee -a gpurun_out/r02_race_check_drop1.txt
timeout 900 python tools/race_check.py --lib tools/ab/libcommet_debug_drop2.so --expect-fail > gpurun_out/r02_race_check_drop2.txt 2>&1; echo "drop2 rc=$?" | tee -a gpurun_out/r02_race_check_drop2.txt
timeout 900 python tools/race_check.py --lib paper_2510_00884_b200/libcommet.so --repeats 10 > gpurun_out/r02_race_check_product.txt 2>&1; echo "product rc=$?" | tee -a gpurun_out/r02_race_check_product.txt
