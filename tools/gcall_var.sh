O=gpurun_out
python tools/time_variants.py default var_ring0 > $O/variants3.jsonl 2>&1
python -m pytest tests -m gpu -x -q > $O/pytest_gpu2.txt 2>&1; tail -2 $O/pytest_gpu2.txt
python bench.py --steps 20 --warmup 5 > $O/bench3.jsonl 2> $O/bench3.err
