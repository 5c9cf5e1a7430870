# quick check after a kernel change: scan / rbi parity, scan path timings, bench
O=gpurun_out
python -m pytest tests/test_gpu_scan.py tests/test_gpu_rbi.py -x -q > $O/quick_pytest.txt 2>&1; tail -2 $O/quick_pytest.txt
python tools/time_scan_paths.py 30 > $O/quick_scan_paths.txt 2>&1
python bench.py --steps 20 --warmup 5 > $O/quick_bench.jsonl 2> $O/quick_bench.err
