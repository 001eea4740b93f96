#!/bin/bash
# The product's radix passes vs CUB SortPairs on 16M pairs (random keys, and the
# C4 tick's own compact keys), with clocks sampled during the runs.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv,noheader -lms 50 > gpurun_out/sc_clocks.csv &
SMI=$!
./scripts/micro/sort_compare > gpurun_out/sort_compare_random.json 2> gpurun_out/sort_compare.err
KX_DUMP_KEYS=/tmp/c4_keys.bin timeout 300 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>> gpurun_out/sort_compare.err
./scripts/micro/sort_compare 16000000 /tmp/c4_keys.bin > gpurun_out/sort_compare_c4.json 2>> gpurun_out/sort_compare.err
kill $SMI
