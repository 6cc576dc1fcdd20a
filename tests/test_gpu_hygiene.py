"""GPU tests of the boundary's promises (include/llama_b200.h conventions):
thread safety of the plan / launch caches under concurrent host threads,
trace counters read after work on a non-blocking stream, and a stager reused
across calls on different streams.  Every result is compared with the oracle."""
import threading

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def llama():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_04284_b200 as m
    return m


# pairs whose plans use different kernels and shared-memory sizes (small and
# wide records, direct variant, word mode, transposes), so concurrent first
# launches race on every launch cache
PAIRS = [(W.PARTICLE7, [40_000], "aos", "soa_mb"), (W.PARTICLE7, [40_000], "aosoa8", "aosoa32"),
         (W.HEP100, [3000], "aos", "soa_mb"), (W.HEP100, [3000], "soa_mb", "aos_aligned"),
         (W.HEP100, [3000], "aos", "aos_aligned"), (W.LISTING1, [200, 96], "aosoa32", "soa_sb"),
         (W.LISTING1, [5000], "soa_mb", "aos_aligned"), (W.PARTICLE7, [64, 64], "aos", "soa_mb")]


def _expected(oracle, schema, ext, a, b, seed):
    so = oracle.mapping_from_spec(schema, ext, W.resolve_spec(a))
    do = oracle.mapping_from_spec(schema, ext, W.resolve_spec(b))
    return oracle.copy(so, oracle.make_view(so, seed), do)


def test_concurrent_host_threads(llama, oracle_mod):
    """8 host threads, each with its own stream and fresh mappings (new plan
    cache entries), copy different pairs at once, several rounds; every
    destination equals the oracle's copy."""
    exp = {j: _expected(oracle_mod, *p, seed=100 + j) for j, p in enumerate(PAIRS)}
    errors = []
    dev = torch.cuda.current_device()

    def worker(j):
        try:
            torch.cuda.set_device(dev)
            schema, ext, a, b = PAIRS[j]
            stream = torch.cuda.Stream()
            for rnd in range(3):
                sm = llama.Mapping.from_spec(schema, ext, W.resolve_spec(a))
                dm = llama.Mapping.from_spec(schema, ext, W.resolve_spec(b))
                if j == len(PAIRS) - 1:
                    dm = dm.with_linearizer("col")  # a transposing copy (k_transpose2d)
                with torch.cuda.stream(stream):
                    sb, db = sm.alloc("cuda"), dm.alloc("cuda")
                    llama.generate(sm, sb, 100 + j, stream=stream)
                    for t in db:
                        t.fill_(0x5A)
                    llama.copy(sm, sb, dm, db, stream=stream)
                stream.synchronize()
                if j == len(PAIRS) - 1:
                    so = oracle_mod.mapping_from_spec(schema, ext, W.resolve_spec(a))
                    do = oracle_mod.mapping_from_spec(schema, ext, W.resolve_spec(b), lin="col")
                    want = oracle_mod.copy(so, oracle_mod.make_view(so, 100 + j), do)
                else:
                    want = exp[j]
                for q, t in enumerate(db):
                    if not np.array_equal(t.cpu().numpy(), want[q]):
                        errors.append((j, rnd, q))
        except Exception as ex:  # reported below
            errors.append((j, repr(ex)))

    threads = [threading.Thread(target=worker, args=(j,)) for j in range(len(PAIRS))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


def test_trace_counters_after_nonblocking_stream(llama, oracle_mod):
    """Counters read right after a traced copy enqueued on a non-blocking
    stream (no caller sync) include that copy (llama_trace_field_hits
    synchronises the counters' device)."""
    n = 1 << 20
    sm = llama.Mapping(W.PARTICLE7, [n], "aos").traced(fields=True)
    dm = llama.Mapping(W.PARTICLE7, [n], "soa_mb")
    sb, db = sm.alloc("cuda"), dm.alloc("cuda")
    llama.generate(sm, sb, 5)
    torch.cuda.synchronize()
    sm.reset_trace()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    for _ in range(4):
        llama.copy(sm, sb, dm, db, stream=s)
    assert sm.field_hits() == [4 * n] * 7


def test_stager_reused_across_streams(llama, oracle_mod):
    """Consecutive staged calls on one stager from different non-blocking
    streams: every reuse of a staging buffer waits for its previous slab, so
    neither copy corrupts the other."""
    n = 300_000
    st = llama.Stager(1 << 20)  # many slabs per call
    outs = []
    for j, (a, b) in enumerate([("aos", "soa_mb"), ("soa_mb", "aosoa8"), ("aosoa8", "aos_aligned")]):
        so = oracle_mod.mapping_from_spec(W.PARTICLE7, [n], W.resolve_spec(a))
        do = oracle_mod.mapping_from_spec(W.PARTICLE7, [n], W.resolve_spec(b))
        src = oracle_mod.make_view(so, 7 + j)
        exp = oracle_mod.copy(so, src, do)
        sm = llama.Mapping.from_spec(W.PARTICLE7, [n], W.resolve_spec(a))
        dm = llama.Mapping.from_spec(W.PARTICLE7, [n], W.resolve_spec(b))
        hs = [torch.from_numpy(x.copy()).pin_memory() for x in src]
        hd = [torch.full((sz,), 0x5A, dtype=torch.uint8).pin_memory() for sz in dm.blob_sizes()]
        llama.copy_staged(st, sm, hs, dm, hd, stream=torch.cuda.Stream())
        outs.append((hd, exp, hs))
    torch.cuda.synchronize()
    for hd, exp, _ in outs:
        for q, t in enumerate(hd):
            assert np.array_equal(t.numpy(), exp[q])
