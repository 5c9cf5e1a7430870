O=gpurun_out
python tools/time_variants.py default var_nosplit default var_nosplit > $O/variants5.jsonl 2>&1
python -m pytest tests/test_gpu_scan.py tests/test_gpu_random_cases.py tests/test_gpu_dist_emulated.py tests/test_gpu_edge_cases.py tests/test_gpu_reduce.py -x -q > $O/q_pytest5.txt 2>&1; tail -2 $O/q_pytest5.txt
