import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
import paper_2106_04284_b200 as llama, workloads as W, oracle
from test_gpu_lin_trace import _pair
KINDS = [("aos", 1, False), ("aos", 1, True), ("soa_mb", 1, False), ("soa_sb", 1, True), ("aosoa", 8, False), ("aosoa", 4, True), ("aosoa", 32, False)]
LINS = [("row", "col"), ("col", "row"), ("row", "morton"), ("morton", "col"), ("col", "morton"), ("morton", "row")]
for schema, ext in ((W.PARTICLE7, [64, 96]), (W.LISTING1, [32, 64])):
    for sk in KINDS:
        for dk in KINDS:
            for lins in LINS:
                e = ext if "morton" not in lins else [64, 64]
                sm = llama.Mapping.from_spec(schema, e, sk, lin=lins[0]); dm = llama.Mapping.from_spec(schema, e, dk, lin=lins[1])
                pl = llama.plan(sm, dm, knobs={"jit": 2})
                try:
                    _pair(llama, oracle, schema, e, sk, lins[0], dk, lins[1], seed=21, paths=("auto",), knobs={"jit": 2})
                except AssertionError as ex:
                    print("FAIL", schema[:10], e, sk, lins, dk, pl, str(ex)[:200], flush=True)
                except Exception as ex:
                    print("ERR", schema[:10], e, sk, lins, dk, pl, str(ex)[:200], flush=True)
                    raise
print("done")
