O=gpurun_out
python tools/time_variants.py default var_ext384 > $O/variants4.jsonl 2>&1
python -m pytest tests/test_gpu_scan.py tests/test_gpu_edge_cases.py tests/test_gpu_random_cases.py -x -q -k "min or max or Min or Max or ext or random" > $O/q_pytest2.txt 2>&1
bash tools/gcall_sanitize.sh
