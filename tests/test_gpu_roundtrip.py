"""GPU round-trip identity (BASELINE north_star: "AoS -> SoA -> AoSoA -> AoS
round-trip identity"; the copy is a bijection between the two mappings'
leaf bytes): a cycle of copies through every mapping kind,
each leg on the planner's path or a forced one, must return the starting
blobs byte for byte. Complements the oracle parity of test_gpu_parity.py with
an invariant that holds at any size, so it also runs at C2's full 16M
records. Destination blobs are pre-filled with garbage so an unwritten byte
cannot pass; the generated source padding is 0 (destination padding is
written 0, reading #12)."""
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

CYCLE = ["aos", "soa_mb", "aosoa8", "aos_aligned", "soa_sb", "aosoa32", "aosoa4", "aos"]


@pytest.fixture(scope="module")
def llama():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_04284_b200 as m
    return m


def _cycle(llama, schema, extents, path=None, seed=5):
    maps = [llama.Mapping.from_spec(W.SCHEMAS[schema], extents, W.resolve_spec(k)) for k in CYCLE]
    start = maps[0].alloc()
    llama.generate(maps[0], start, seed)
    cur = start
    for a, b in zip(maps, maps[1:]):
        nxt = b.alloc()
        for t in nxt:
            t.fill_(0xA5)
        llama.copy(a, cur, b, nxt, path=path)
        cur = nxt
    torch.cuda.synchronize()
    # only the view's bytes: an empty blob is a 16-byte placeholder outside the view
    return all(torch.equal(x[:z], y[:z]) for x, y, z in zip(start, cur, maps[0].blob_sizes()))


@pytest.mark.parametrize("schema,n", [("particle7", 4096 + 37), ("listing1", 1000 + 13),
                                      ("hep100", 640 + 21), ("particle7", 0), ("particle7", 1)])
@pytest.mark.parametrize("path", [None, "naive"])
def test_cycle_identity_ragged(llama, schema, n, path):
    assert _cycle(llama, schema, (n,), path=path)


def test_cycle_identity_2d(llama):
    assert _cycle(llama, "listing1", (67, 93))


def test_cycle_identity_c2_full(llama):
    n = W.C2["extents"][0]  # 16,777,216 Particle7 records, the bench workload
    assert _cycle(llama, "particle7", (n,))
