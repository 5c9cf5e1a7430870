# ncu --set full of the MAT2 return sweep alone (second scan_apply launch of tools/prof_config2.py), exported as text
O=gpurun_out
ncu --set full --import-source on --clock-control none -k regex:scan_apply --launch-skip 1 --launch-count 1 -o /tmp/mat2 python tools/prof_config2.py > $O/mat2.log 2>&1
ncu -i /tmp/mat2.ncu-rep --page details > $O/r02_ncu_full_apply_mat2_final.txt 2>&1
ncu -i /tmp/mat2.ncu-rep --page raw --csv > /tmp/mat2_raw.csv 2>&1
python tools/ncu_stalls.py /tmp/mat2_raw.csv > $O/r02_ncu_apply_mat2_final_stalls.txt 2>&1
ncu -i /tmp/mat2.ncu-rep --page source --csv --print-source sass > /tmp/mat2_src.csv 2>&1
python tools/ncu_hot_sass.py /tmp/mat2_src.csv 60 > $O/r02_ncu_apply_mat2_final_hot_sass.txt 2>&1
