#!/usr/bin/env python
"""One n-body move per layout (SoA MB, AoS, AoSoA32, split_p7) at the bench's 256Mi particles
(W.NBODY_MOVE_N), for ncu captures (tools/traffic_from_ncu.py ...:MOVE)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_04284_b200 as llama  # noqa: E402
import workloads as W  # noqa: E402

n = W.NBODY_MOVE_N
for name in ("soa_mb", "aos", "aosoa32", "split_p7"):
    m = llama.Mapping.from_spec(W.PARTICLE7, [n], W.resolve_spec(name))
    b = m.alloc("cuda")
    for t in b:
        t.zero_()
    print(name, llama.nbody_move(m, b, 1e-4))
    torch.cuda.synchronize()
    del b
