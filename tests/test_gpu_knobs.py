"""Tuning knobs at extreme values (llama_copy_options.knobs, include/llama_b200.h):
every knob the planner takes from the caller either yields a plan whose copy is
still byte-exact against the oracle, or is refused before any launch
(UNSUPPORTED / INVALID_ARGUMENT from the planner, the forced path then
skipped) -- never a failed launch (LLAMA_ERR_CUDA).  The ablation knob is
excluded: it skips the move program by design."""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

VALUES = [0, 1, 3, 1 << 20, 1 << 40]
# (schema, extents, src spec, src lin, dst spec, dst lin, forced paths besides auto)
CASES = [
    ("particle7", [1000], ("aos", 1, False), "row", ("soa_mb", 1, False), "row", ("permute", "naive")),
    ("particle7", [1000], ("soa_mb", 1, False), "row", ("soa_mb", 1, False), "row", ("blobcopy", "run")),
    ("hep100", [300], ("aos", 1, False), "row", ("soa_mb", 1, False), "row", ("permute",)),
    ("hep100", [300], ("soa_mb", 1, False), "row", ("aos", 1, True), "row", ("permute",)),
    ("particle7", [64, 64], ("aos", 1, False), "row", ("soa_mb", 1, False), "col", ("transpose",)),
    ("particle7", [64, 64], ("aos", 1, False), "row", ("aos", 1, False), "col", ("transpose",)),
]
_EXP = {}


@pytest.fixture(scope="module")
def llama():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_04284_b200 as m
    return m


def _case(llama, oracle, i):
    schema, ext, ss, sl, ds, dl, paths = CASES[i]
    sch = W.SCHEMAS[schema]
    sm = llama.Mapping.from_spec(sch, ext, ss, lin=sl)
    dm = llama.Mapping.from_spec(sch, ext, ds, lin=dl)
    if i not in _EXP:
        so = oracle.mapping_from_spec(sch, ext, ss, lin=sl)
        do = oracle.mapping_from_spec(sch, ext, ds, lin=dl)
        src = oracle.make_view(so, 5 + i, pad_fill=0xCD)
        _EXP[i] = oracle.copy(so, src, do)
    sb = sm.alloc("cuda")
    llama.generate(sm, sb, 5 + i, pad_byte=0xCD)
    return sm, sb, dm, _EXP[i], paths


@pytest.mark.parametrize("knob", [k for k in __import__("paper_2106_04284_b200").KNOBS if k != "jit_ablate"])
def test_knob_extremes(llama, oracle_mod, knob):
    for i in range(len(CASES)):
        sm, sb, dm, exp, paths = _case(llama, oracle_mod, i)
        for v in VALUES:
            knobs = {knob: v, "jit": 2} if knob.startswith("jit_") else {knob: v}
            for path in ("auto",) + paths:
                try:
                    llama.plan(sm, dm, path=None if path == "auto" else path, knobs=knobs)
                except llama.LlamaError as e:
                    assert path != "auto", (knob, v, i, str(e))
                    continue
                db = dm.alloc("cuda")
                for t in db:
                    t.fill_(0x5A)
                try:
                    llama.copy(sm, sb, dm, db, path=None if path == "auto" else path, knobs=knobs)
                except llama.LlamaError as e:
                    raise AssertionError(f"knob {knob}={v} case {i} path {path}: the plan was accepted but the copy "
                                         f"failed: {e}")
                torch.cuda.synchronize()
                for j, t in enumerate(db):
                    assert np.array_equal(t.cpu().numpy(), exp[j]), (knob, v, i, path, j)
