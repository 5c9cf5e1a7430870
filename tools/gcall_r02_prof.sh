# round-2 profiling pass: ncu captures exported to text on the box (the .ncu-rep
# files are too large to bring back), PCIe probe, e2e bench
set -x
O=gpurun_out
python tools/pcie_probe.py > $O/pcie.jsonl 2>&1
cap() {  # name, kernel regex, count, script
  ncu --set full --import-source on --clock-control none -k regex:$2 -c $3 -o /tmp/$1 python $4 > $O/$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page details > $O/$1_details.txt 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > /tmp/$1_raw.csv 2>&1
  python tools/ncu_stalls.py /tmp/$1_raw.csv > $O/$1_stalls.txt 2>&1
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > /tmp/$1_src.csv 2>&1
  python tools/ncu_hot_sass.py /tmp/$1_src.csv > $O/$1_hot.txt 2>&1
}
cap r02_ncu_config2_apply scan_apply 4 tools/prof_config2.py
cap r02_ncu_config2_reduce scan_reduce 2 tools/prof_config2.py
cap r02_ncu_rbi_fwd_smem_log rbi_fwd_smem_log 1 tools/prof_rbi_mul.py
cap r02_ncu_rbi_bwd_mul rbi_bwd_map 1 tools/prof_rbi_mul.py
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/prof_rbi_mul.py > $O/rbi_mul_launches.csv 2> $O/ncu5.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Ipaper_2202_10297_b200/csrc -o /tmp/exp_rbi_fwd tools/exp_rbi_fwd.cu && /tmp/exp_rbi_fwd > $O/exp_rbi_fwd.jsonl 2>&1
python bench.py --steps 20 --warmup 5 > $O/bench_e2e16.jsonl 2> $O/bench_e2e16.err
du -sh $O
