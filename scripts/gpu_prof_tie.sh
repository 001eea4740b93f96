export PER_POOL=2000000
bash scripts/gpu_ncu_one.sh "k_tie_runs|k_tie_fix_small" prof_tie 2 2
bash scripts/gpu_ncu_one.sh "k_onesweep_pass" prof_sweep 5 2
