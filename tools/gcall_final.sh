# final check of the committed build: the GPU suite, smoke(), the default bench
O=gpurun_out
python -m pytest tests -m gpu -x -q > $O/pytest_gpu_final.txt 2>&1; tail -2 $O/pytest_gpu_final.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke_final.txt 2>&1; tail -2 $O/smoke_final.txt
python bench.py > $O/bench_final2.jsonl 2> $O/bench_final2.err
