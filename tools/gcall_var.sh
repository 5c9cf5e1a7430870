O=gpurun_out
python tools/time_variants.py default var_minb5 var_minb6 default var_minb5 var_minb6 > $O/variants10.jsonl 2>&1
