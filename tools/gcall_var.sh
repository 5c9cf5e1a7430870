O=gpurun_out
TV_SCAN_ADD=1 python tools/time_variants.py default var_m3 var_m6 default var_m3 var_m6 > $O/variants12.jsonl 2>&1
