O=gpurun_out
python tools/time_variants.py default var_bwd1 default var_bwd1 > $O/variants9.jsonl 2>&1
python -m pytest tests/test_gpu_rbi.py tests/test_gpu_dist_emulated.py tests/test_gpu_edge_cases.py -x -q > $O/q_pytest9.txt 2>&1; tail -2 $O/q_pytest9.txt
