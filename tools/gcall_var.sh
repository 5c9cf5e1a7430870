O=gpurun_out
python tools/time_variants.py default var_sc2 default var_sc2 > $O/variants11.jsonl 2>&1
VJP_X=1 python -c "
import sys; sys.path.insert(0,'.')
import paper_2202_10297_b200 as vjp, os
vjp.LIB_PATH=os.path.join('paper_2202_10297_b200','_lib','var_sc2.so')
import pytest
sys.exit(pytest.main(['tests/test_gpu_scan.py','-x','-q','-k','linrec']))
" > $O/q_pytest11.txt 2>&1; tail -2 $O/q_pytest11.txt
