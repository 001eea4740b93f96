set -u
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_dispatch_lanes" -s 2 -c 1 \
   -o gpurun_out/prof_disp -f python scripts/dispatch_probe.py 2000000 2 > gpurun_out/ncu_disp.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_disp.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_topk_sort|k_tie_runs|k_keygen|k_topk_hist" -s 8 -c 6 \
   -o gpurun_out/prof_misc -f python scripts/dispatch_probe.py 2000000 2 > gpurun_out/ncu_misc.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_misc.log
