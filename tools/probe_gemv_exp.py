"""probe_gemv.py with the trace build's experiment switch applied (PPSD_TC_EXP bits:
1 = no weight copies, 2 = no operand builds; results are wrong, times are the point).

    PPSD_TC_EXP=3 PPSD_LIB=<trace build>/libppsd.so python tools/probe_gemv_exp.py 20 qkv 1,-16
"""
import os, sys
sys.path.insert(0, os.getcwd())
sys.argv = ["probe_gemv.py"] + sys.argv[1:]
import paper_2509_19368_b200 as ppsd
from paper_2509_19368_b200 import _lib
import tools.probe_gemv as pg
orig = ppsd.engine_for
def ef(*a, **k):
    e = orig(*a, **k)
    _lib.check(_lib.lib().ppsd_debug_tc_trace(0, None), "exp")
    return e
ppsd.engine_for = ef
pg.ppsd.engine_for = ef
pg.main()
