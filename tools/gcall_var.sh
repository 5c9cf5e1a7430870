O=gpurun_out
python tools/time_variants.py default var_noapplyfused default var_noapplyfused > $O/variants8.jsonl 2>&1
python -m pytest tests/test_gpu_scan.py tests/test_gpu_random_cases.py tests/test_gpu_dist_emulated.py tests/test_gpu_edge_cases.py tests/test_gpu_reduce.py tests/test_gpu_cyclic.py -x -q > $O/q_pytest8.txt 2>&1; tail -2 $O/q_pytest8.txt
