#!/usr/bin/env python
"""One n-body move per layout (AoS, SoA MB, AoSoA32) on 64Mi particles, for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_04284_b200 as llama  # noqa: E402
import workloads as W  # noqa: E402

n = 1 << 26
for name in ("soa_mb", "aos", "aosoa32"):
    m = llama.Mapping.from_spec(W.PARTICLE7, [n], W.resolve_spec(name))
    b = m.alloc("cuda")
    for t in b:
        t.zero_()
    print(name, llama.nbody_move(m, b, 1e-4))
    torch.cuda.synchronize()
    del b
