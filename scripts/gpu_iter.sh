#!/bin/bash
# Iteration: GPU parity tests, short bench, ncu launch list.
bash scripts/gpu_quick.sh
bash scripts/gpu_launches.sh
