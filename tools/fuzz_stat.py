import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np, pytest
src=open('tests/test_gpu_fuzz.py').read()
exec(src.replace("pytestmark = pytest.mark.gpu",""))
from paper_2510_12739_b200 import plan as P
cnt={}
for s in range(48):
    g,x=_random_graph(1000+s)
    row=[]
    for prec in ("bf16","bf16x3"):
        try: P.Plan(g,prec); row.append(prec)
        except P.CnrxUnsupported as e: row.append("-"+str(e)[:60])
    print(s, row)
