"""CPU-side tests of the C-ABI library: it loads, exports every symbol the
header declares, and its host-side descriptor (the AoSoA normal form,
mapping.cpp) agrees with the oracle's independent per-kind formulas
(oracle.c) exhaustively on small extents (SURVEY P11 brute force).  Validation
errors are raised before any device work, so no GPU is needed here."""
import ctypes
import os
import re

import numpy as np
import pytest

import workloads as W
from conftest import ROOT

llama = pytest.importorskip("paper_2106_04284_b200")


def test_exports_every_declared_symbol():
    with open(os.path.join(ROOT, "include", "llama_b200.h")) as f:
        text = f.read()
    declared = set(re.findall(r"\b(llama_[a-z_]+)\s*\(", text))
    assert declared == set(llama.EXPORTS)
    lib = llama.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert "sm_100a" in llama.version()


def test_library_reads_no_environment():
    """A plan depends only on the mappings and the explicit options (knobs):
    no source of the library reads the environment."""
    csrc = os.path.join(ROOT, "paper_2106_04284_b200", "csrc")
    for name in os.listdir(csrc):
        with open(os.path.join(csrc, name)) as f:
            assert "getenv" not in f.read(), name


def test_knob_names_match_header():
    with open(os.path.join(ROOT, "include", "llama_b200.h")) as f:
        text = f.read()
    body = text[text.index("LLAMA_KNOB_TILE_BYTES"):text.index("LLAMA_KNOB_COUNT")]
    names = [n.lower() for n in re.findall(r"LLAMA_KNOB_([A-Z0-9_]+)", body)]
    assert names == llama.KNOBS


def test_bad_knob_name_is_rejected():
    m = llama.Mapping(W.PARTICLE7, [64], "aos")
    with pytest.raises(ValueError):
        llama.plan(m, m, knobs={"no_such_knob": 1})


def test_knobs_change_the_plan_and_key_the_cache():
    """Explicit knobs reach the planner, and plans with different knobs are
    cached separately (host only: llama_plan does no device work)."""
    a = llama.Mapping(W.PARTICLE7, [1 << 20], "aos")
    b = llama.Mapping(W.PARTICLE7, [1 << 20], "soa_mb")
    base = llama.plan(a, b)
    small = llama.plan(a, b, knobs={"tile_bytes": 16 * 1024})
    assert small["tile_records"] < base["tile_records"]
    assert llama.plan(a, b)["tile_records"] == base["tile_records"]
    assert not llama.plan(a, b, knobs={"no_tma": 1})["tma"]
    h = llama.Mapping(W.HEP100, [4096], "aos", 1, True)
    hs = llama.Mapping(W.HEP100, [4096], "soa_mb")
    assert llama.plan(h, hs)["jit"]
    assert llama.plan(h, hs, knobs={"jit": 0})["direct"]
    assert not llama.plan(h, hs, knobs={"jit": 0, "direct": 0})["direct"]


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", llama.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


KINDS = [("aos", 1, False), ("aos", 1, True), ("soa_sb", 1, False), ("soa_sb", 1, True), ("soa_mb", 1, False),
         ("aosoa", 1, False), ("aosoa", 2, False), ("aosoa", 3, False), ("aosoa", 4, False), ("aosoa", 8, True),
         ("aosoa", 32, False)]


@pytest.mark.parametrize("schema", [W.LISTING1, W.PARTICLE7, W.OUTER, W.HEP100, W.VEC])
@pytest.mark.parametrize("ext", [[1], [5], [33], [4, 3], [2, 3, 5]])
def test_descriptor_matches_oracle(oracle_mod, schema, ext):
    n = int(np.prod(ext))
    for kind, L, aligned in KINDS + [("aosoa", n, False)]:
        m = llama.Mapping(schema, ext, kind, L, aligned)
        o = oracle_mod.Mapping(schema, ext, kind, L, aligned)
        assert m.blob_sizes() == o.blob_sizes()
        assert m.record_count == o.record_count == n
        assert m.leaf_count == o.n_leaves
        for flat in range(n):
            idx = list(np.unravel_index(flat, ext))
            for k in range(o.n_leaves):
                assert m.blob_nr_and_offset([int(x) for x in idx], k) == o.addr(flat, k)


def test_big_extents_blob_sizes(oracle_mod):
    for cfg in W.CONFIGS.values():
        schema = W.SCHEMAS[cfg["schema"]]
        for a, b in cfg["pairs"]:
            for name in (a, b):
                kind, L, al = W.MAPPINGS[name]
                m = llama.Mapping(schema, cfg["extents"], kind, L, al)
                o = oracle_mod.Mapping(schema, cfg["extents"], kind, L, al)
                assert m.blob_sizes() == o.blob_sizes()


def test_schema_parser_matches_oracle(oracle_mod):
    for schema in [W.LISTING1, W.HEP100, W.OUTER, "R{a:f32[2][3],b{c:bool[2],d:u16}}", "f64"]:
        m = llama.Mapping(schema, [3], "aos")
        sizes = [{0: 1, 1: 1, 2: 1, 3: 2, 4: 2, 5: 4, 6: 4, 7: 8, 8: 8, 9: 4, 10: 8}[t] for t in m.leaf_types()]
        assert sizes == oracle_mod.leaf_sizes(schema)
    for bad in ["R{a:f16}", "R{a:f32,a:f32}", "R{a:f32[0]}", "R{", "R{a:f32}}"]:
        with pytest.raises(llama.LlamaError) as e:
            llama.Mapping(bad, [3], "aos")
        assert e.value.status == -1


def test_mapping_errors():
    with pytest.raises(llama.LlamaError) as e:
        llama.Mapping(W.VEC, [-1], "aos")
    assert e.value.status == -1
    with pytest.raises(llama.LlamaError) as e:
        llama.Mapping(W.VEC, [4], "aosoa", lanes=0)
    assert e.value.status == -1
    big = "R{" + ",".join(f"f{j}:u8" for j in range(200)) + "}"
    with pytest.raises(llama.LlamaError) as e:
        llama.Mapping(big, [4], "aos")
    assert e.value.status == -4
    m = llama.Mapping(W.VEC, [4, 3], "aos")
    with pytest.raises(llama.LlamaError):
        m.blob_nr_and_offset([4, 0], 0)
    with pytest.raises(llama.LlamaError):
        m.blob_nr_and_offset([0, 0], 2)


def _copy_raw(src, sp, dst, dp):
    lib = llama.lib()
    a = (ctypes.c_void_p * max(1, len(sp)))(*sp)
    b = (ctypes.c_void_p * max(1, len(dp)))(*dp)
    rc = lib.llama_copy(src.handle, a, dst.handle, b, None)
    return rc, lib.llama_last_error_message().decode()


def test_copy_validation_errors_are_synchronous():
    """S:484-486 and the ABI's validation rules; all rejected before launch."""
    a = llama.Mapping(W.LISTING1, [64], "aos")
    b = llama.Mapping(W.LISTING1, [64], "soa_mb")
    rc, _ = _copy_raw(a, [0x10000], llama.Mapping(W.LISTING1, [65], "aos"), [0x90000])
    assert rc == -2
    rc, _ = _copy_raw(a, [0x10000], llama.Mapping(W.VEC, [64], "aos"), [0x90000])
    assert rc == -3
    rc, msg = _copy_raw(a, [0x10008], b, [0x100000 + 0x1000 * j for j in range(7)])
    assert rc == -5 and "src_blobs[0]" in msg
    rc, _ = _copy_raw(a, [0x10000], b, [0x100000 + 0x1000 * j for j in range(6)] + [0])
    assert rc == -1
    # overlapping src/dst (in-situ copies are out of scope)
    rc, _ = _copy_raw(a, [0x10000], b, [0x10000 + 0x100] + [0x100000 + 0x1000 * j for j in range(6)])
    assert rc == -6
    # overlapping destination blobs
    rc, _ = _copy_raw(a, [0x10000], b, [0x100000] * 7)
    assert rc == -6
    lib = llama.lib()
    assert lib.llama_copy(None, None, None, None, None) == -1
    assert lib.llama_status_string(-6) == b"LLAMA_ERR_OVERLAP"


def _plan(src_name, dst_name, schema=W.PARTICLE7, ext=(16_777_216,)):
    s = llama.Mapping(schema, ext, *W.MAPPINGS[src_name])
    d = llama.Mapping(schema, ext, *W.MAPPINGS[dst_name])
    return llama.plan(s, d)


def test_planner_choices_c2():
    """Every C2 pair -> the warp-specialised TMA permute, which on B200 beats
    the bulk blob copy on identities and the direct run copy on pairs
    that share >= 16 B runs; both stay available as forced paths."""
    for name in ("aos", "soa_mb", "aosoa8"):
        s = llama.Mapping(W.PARTICLE7, (1000,), *W.MAPPINGS[name])
        d = llama.Mapping(W.PARTICLE7, (1000,), *W.MAPPINGS[name])
        assert llama.plan(s, d, path="blobcopy")["path"] == "blobcopy"
    assert _plan("soa_mb", "soa_mb", W.HEP100, (1 << 20,))["path"] == "blobcopy"  # many-leaf SoA identity
    for a, b in [("aos", "aos"), ("soa_mb", "soa_mb"), ("aos", "soa_mb"), ("soa_mb", "aos"), ("aos", "aosoa8"), ("aosoa32", "aos"),
                 ("aosoa8", "aosoa32"), ("soa_mb", "aosoa8"), ("aosoa32", "soa_mb")]:
        p = _plan(a, b)
        assert p["path"] == "permute" and p["tma"] and p["tile_records"] % 32 == 0
    for a, b in [("aosoa8", "aosoa32"), ("soa_mb", "aosoa8"), ("aosoa32", "soa_mb")]:
        s = llama.Mapping(W.PARTICLE7, (1024,), *W.MAPPINGS[a])
        d = llama.Mapping(W.PARTICLE7, (1024,), *W.MAPPINGS[b])
        assert llama.plan(s, d, path="run")["path"] == "run"
    assert _plan("aosoa32", "soa_sb", W.LISTING1, (8192, 8192))["path"] == "permute"  # C4
    for a, b in W.C3["pairs"]:
        p = _plan(a, b, W.HEP100, (67_108_864,))
        assert p["path"] == "permute", (a, b, p)
    assert _plan("aos", "soa_mb", ext=(4096,))["path"] == "permute"  # C1


def test_planner_forced_paths():
    s = llama.Mapping(W.PARTICLE7, [1000], "aos")
    d = llama.Mapping(W.PARTICLE7, [1000], "soa_mb")
    assert llama.plan(s, d, path="naive")["path"] == "naive"
    with pytest.raises(llama.LlamaError) as e:
        llama.plan(s, d, path="run")
    assert e.value.status == -4
    with pytest.raises(llama.LlamaError):
        llama.plan(s, d, path="permute", tile_records=48)
    assert llama.plan(s, d, path="permute", tile_records=64)["tile_records"] == 64


# ------------------------------------------------------------ One / Split (f1)
SPLIT_NAMES = sorted(W.SPLITS)


@pytest.mark.parametrize("name", SPLIT_NAMES + ["one"])
@pytest.mark.parametrize("ext", [[1], [5], [33], [4, 3]])
def test_split_one_descriptor_matches_oracle(oracle_mod, name, ext):
    schema = W.SCHEMAS[W.SPLITS[name][0]] if name in W.SPLITS else W.LISTING1
    spec = W.resolve_spec(name)
    m = llama.Mapping.from_spec(schema, ext, spec)
    o = oracle_mod.mapping_from_spec(schema, ext, spec)
    assert m.blob_sizes() == o.blob_sizes()
    assert m.leaf_types() == llama.Mapping(schema, ext).leaf_types()
    n = int(np.prod(ext))
    for flat in range(n):
        idx = [int(x) for x in np.unravel_index(flat, ext)]
        for k in range(o.n_leaves):
            assert m.blob_nr_and_offset(idx, k) == o.addr(flat, k)


def test_split_errors_and_plans():
    sizes = llama.Mapping(W.LISTING1, [4]).leaf_types()
    a = llama.Mapping(sizes[:2], [4], "soa_mb")
    b = llama.Mapping(sizes[2:], [4], "aos")
    llama.Mapping.split(a, b, [0, 1])
    with pytest.raises(llama.LlamaError, match="INVALID_ARGUMENT"):
        llama.Mapping.split(a, b, [1, 0])
    with pytest.raises(llama.LlamaError, match="INVALID_ARGUMENT"):
        llama.Mapping.split(a, b, [0])
    with pytest.raises(llama.LlamaError, match="INVALID_ARGUMENT"):
        llama.Mapping.split(a, llama.Mapping(sizes[2:], [5], "aos"), [0, 1])
    aos = llama.Mapping(W.LISTING1, [4])
    one = llama.Mapping(W.LISTING1, [4], "one")
    mc = llama.Mapping.from_spec(W.LISTING1, [4], W.resolve_spec("mapping_c"))
    # a destination that maps several records onto one place is rejected (reading #24)
    for dst in (one, mc):
        with pytest.raises(llama.LlamaError, match="UNSUPPORTED"):
            llama.plan(aos, dst)
    assert llama.plan(one, aos)["path"] == "naive"
    assert llama.plan(mc, aos)["path"] == "naive"
    one1 = llama.Mapping(W.LISTING1, [1], "one")
    llama.plan(llama.Mapping(W.LISTING1, [1]), one1)  # one record: no collision
    sp = llama.Mapping.from_spec(W.LISTING1, [4], W.resolve_spec("split_pos"))
    assert llama.plan(sp, sp, path="blobcopy")["path"] == "blobcopy"
    # splits whose parts all spread records over blobs take the tile permute (parts per side)
    big = [1 << 20]
    for name, other in (("split_p7", "aos"), ("split_p7", "soa_mb"), ("split_pos", "aos_aligned"),
                        ("split_hep", "aos")):
        schema = W.SCHEMAS[W.SPLITS[name][0]]
        a = llama.Mapping.from_spec(schema, big, W.resolve_spec(name))
        b = llama.Mapping(schema, big, *W.MAPPINGS[other])
        assert llama.plan(a, b)["path"] == "permute", (name, other)
        assert llama.plan(b, a)["path"] == "permute", (other, name)


# ------------------------------------------------------- linearisations (f4)
@pytest.mark.parametrize("lin,ext", [("col", [4, 3]), ("col", [2, 3, 5]), ("morton", [4, 4]), ("morton", [2, 2, 2])])
@pytest.mark.parametrize("name", ["aos", "soa_sb", "aosoa4", "split_pos"])
def test_linearized_descriptor_matches_oracle(oracle_mod, lin, ext, name):
    spec = W.resolve_spec(name) if name != "aosoa4" else ("aosoa", 4, False)
    m = llama.Mapping.from_spec(W.LISTING1, ext, spec, lin=lin)
    o = oracle_mod.mapping_from_spec(W.LISTING1, ext, spec, lin=lin)
    assert m.blob_sizes() == o.blob_sizes()
    for flat in range(int(np.prod(ext))):
        idx = [int(x) for x in np.unravel_index(flat, ext)]
        for k in range(o.n_leaves):
            assert m.blob_nr_and_offset(idx, k) == o.addr(flat, k)


def test_linearizer_errors_and_plans():
    row = llama.Mapping(W.PARTICLE7, [64, 64])
    col = row.with_linearizer("col")
    assert llama.plan(row, col)["path"] == "transpose"  # a transposing copy: 32x32-record tiles
    assert llama.plan(row, col, path="naive")["path"] == "naive"
    with pytest.raises(llama.LlamaError, match="UNSUPPORTED"):
        llama.plan(row, llama.Mapping(W.PARTICLE7, [64, 64], "soa_mb"), path="transpose")

    with pytest.raises(llama.LlamaError, match="UNSUPPORTED"):
        llama.plan(row, col, path="permute")
    soa_col = llama.Mapping(W.PARTICLE7, [64, 64], "soa_mb").with_linearizer("col")
    assert llama.plan(col, soa_col)["path"] == "permute"  # equal storage orders: every path
    with pytest.raises(llama.LlamaError, match="INVALID_ARGUMENT"):
        llama.Mapping(W.PARTICLE7, [64, 32]).with_linearizer("morton")
    with pytest.raises(llama.LlamaError, match="INVALID_ARGUMENT"):
        llama.Mapping(W.PARTICLE7, [48, 48]).with_linearizer("morton")
    sizes = llama.Mapping(W.LISTING1, [4]).leaf_types()
    a = llama.Mapping(sizes[:2], [4], "soa_mb").with_linearizer("col")
    b = llama.Mapping(sizes[2:], [4], "aos")
    with pytest.raises(llama.LlamaError, match="INVALID_ARGUMENT"):
        llama.Mapping.split(a, b, [0, 1])


def _jit_cases():
    m = {k: llama.Mapping(W.HEP100, [1 << 20], *W.MAPPINGS[k]) for k in ("aos", "aos_aligned", "soa_mb")}
    cases = [(f"hep_{a}_{b}", m[a], m[b], None) for a in m for b in m if a != b]
    l1 = {k: llama.Mapping(W.LISTING1, [1 << 20], *W.MAPPINGS[k]) for k in ("aos", "soa_mb", "aosoa32", "soa_sb")}
    cases += [(f"l1_{a}_{b}", l1[a], l1[b], {"jit": 2}) for a, b in
              [("aos", "soa_mb"), ("soa_mb", "aos"), ("aosoa32", "soa_sb"), ("aosoa32", "aos")]]
    for schema, a, b in [(W.LISTING1, "aos", "split_pos"), (W.HEP100, "aos", "split_hep"), (W.HEP100, "split_hep", "soa_mb"),
                         (W.PARTICLE7, "split_p7", "aos")]:
        cases.append((f"split_{a}_{b}", llama.Mapping.from_spec(schema, [1 << 20], W.resolve_spec(a)),
                      llama.Mapping.from_spec(schema, [1 << 20], W.resolve_spec(b)), None))
    for a, b in [("aos_aligned", "split_pos"), ("split_pos", "aos_aligned")]:  # padded images (2-word chunk tables)
        cases.append((f"pad_{a}_{b}", llama.Mapping.from_spec(W.LISTING1, [1 << 20], W.resolve_spec(a)),
                      llama.Mapping.from_spec(W.LISTING1, [1 << 20], W.resolve_spec(b)), None))
    return cases


def test_jit_transpose_block_chosen():
    """Block programs are the default for transposes into SoA destinations
    (a Morton source's runs are padded in them), per-record programs into
    AoS images."""
    for sk, sl, dk, dl, blk in [("soa_mb", "col", "soa_mb", "row", 1), ("aos", "row", "soa_mb", "col", 1),
                                ("aos", "row", "aos", "col", 0), ("soa_mb", "morton", "soa_mb", "row", 1)]:
        sm = llama.Mapping.from_spec(W.PARTICLE7, [256, 256], (sk, 1, False), lin=sl)
        dm = llama.Mapping.from_spec(W.PARTICLE7, [256, 256], (dk, 1, False), lin=dl)
        assert llama.plan(sm, dm)["jit"]
        assert f"#define LLB_BLOCK {blk}" in llama.plan_source(sm, dm), (sk, sl, dk, dl)


def test_jit_padded_image_decision():
    """Knob jit_pad: Listing-1 aligned records (32 B, groups of 4 -> 128-byte
    group stride) get padded images by default, moved through 2-word chunk
    tables; jit_pad=0 keeps the TMA op; HEP100 aligned (480-byte stride) is
    padded only under jit_pad=2."""
    al = llama.Mapping.from_spec(W.LISTING1, [1 << 20], W.resolve_spec("aos_aligned"))
    sp = llama.Mapping.from_spec(W.LISTING1, [1 << 20], W.resolve_spec("split_pos"))
    src = llama.plan_source(al, sp)
    assert "#define LLB_CW 2u" in src and "#define LLB_DCW 1u" in src and "r * 144u" in src
    src = llama.plan_source(sp, al)
    assert "#define LLB_CW 1u" in src and "#define LLB_DCW 2u" in src and "dgs[" in src
    src = llama.plan_source(al, sp, knobs={"jit_pad": 0})
    assert "#define LLB_CW 1u" in src and "r * 144u" not in src
    h = {k: llama.Mapping(W.HEP100, [1 << 16], *W.MAPPINGS[k]) for k in ("aos_aligned", "soa_mb")}
    assert "#define LLB_CW 1u" in llama.plan_source(h["aos_aligned"], h["soa_mb"])
    assert "#define LLB_CW 2u" in llama.plan_source(h["aos_aligned"], h["soa_mb"], knobs={"jit_pad": 2})


def test_jit_plans_compile_without_spills():
    """The plan-time specialised kernels of the C3 pairs, Listing-1 pairs (odd
    record strides: 4-record groups) and splits compile on the host (NVRTC needs
    no GPU) and their generated source, compiled again by ptxas, spills
    nothing."""
    import subprocess
    import tempfile
    with tempfile.TemporaryDirectory() as tmp:
        for name, sm, dm, knobs in _jit_cases():
            pl = llama.plan(sm, dm, knobs=knobs)
            assert pl["jit"] and pl["path"] == "permute", (name, pl)
            src = llama.plan_source(sm, dm, knobs=knobs)
            assert "llb_jit_permute" in src
            fn = os.path.join(tmp, name + ".cu")
            with open(fn, "w") as f:
                f.write(src)
            r = subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-cubin",
                                "-std=c++17", "-Xptxas", "-v", "-o", fn + ".cubin", fn], capture_output=True, text=True)
            assert r.returncode == 0, r.stderr[-2000:]
            assert "0 bytes spill stores, 0 bytes spill loads" in r.stderr, (name, r.stderr[-600:])


def test_wide_transpose_plans():
    """HEP100 transposing copies (380 / 480-byte records, too wide for the JIT
    transpose's TY x 32 tiles) take the wide kernel: an AoS side is an image
    side, tiles of 128 records with 32 along an element-wise side's order
    (64 when two images exceed 64 KB), 32 x 32 between element-wise sides;
    Morton tiles are 2^a x 2^a or 2^a x 2^(a+1); knob wide=0 -> naive."""
    def pl(a, sl, b, dl, ext=(1024, 1024), knobs=None):
        sm = llama.Mapping.from_spec(W.HEP100, list(ext), W.resolve_spec(a), lin=sl)
        dm = llama.Mapping.from_spec(W.HEP100, list(ext), W.resolve_spec(b), lin=dl)
        return llama.plan(sm, dm, knobs=knobs)
    p = pl("aos", "row", "soa_mb", "col")
    assert p["path"] == "transpose" and p["wide"] and p["tile_records"] == 128 and p["moves"] == 0
    assert pl("soa_mb", "col", "aos_aligned", "row")["moves"] == 1
    p = pl("aos", "row", "aos_aligned", "col", knobs={"jit": 0})
    assert p["moves"] == 2 and p["tile_records"] == 64
    p = pl("aos", "row", "aos_aligned", "col")  # the JIT transpose with 4-row tiles (per-record programs)
    assert p["jit"] and p["tile_records"] == 128
    assert pl("aos", "row", "aos", "morton")["moves"] == 3
    assert pl("aos_aligned", "row", "aos_aligned", "col")["moves"] == 2  # padding: never copied from the source
    p = pl("soa_mb", "row", "soa_sb", "col")
    assert p["moves"] == 4 and p["tile_records"] == 1024
    assert pl("soa_mb", "morton", "soa_sb", "row", ext=(16, 16))["path"] == "naive"
    assert pl("aos", "morton", "soa_sb", "row", ext=(4, 4))["tile_records"] == 16
    assert pl("aos", "row", "soa_mb", "col", knobs={"wide": 0})["path"] == "naive"
    small = llama.Mapping.from_spec(W.PARTICLE7, [64, 64], W.resolve_spec("aos"), lin="row")
    smallc = llama.Mapping.from_spec(W.PARTICLE7, [64, 64], W.resolve_spec("soa_mb"), lin="col")
    assert not llama.plan(small, smallc)["wide"] and llama.plan(small, smallc, knobs={"wide": 2})["wide"]


def test_jit_permute_scan_rules():
    """The JIT permute rules from the knob scan: AoS-like
    images on both sides take 2 source stages, 256-record tiles without
    record groups; packed misaligned AoS into all-SoA 4 stages; record groups
    into all-SoA store from registers (soa_tma 0)."""
    def src(schema, n, a, b, knobs=None):
        sm = llama.Mapping(schema, [n], *W.MAPPINGS[a])
        dm = llama.Mapping(schema, [n], *W.MAPPINGS[b])
        return llama.plan_source(sm, dm, knobs=knobs)
    s = src(W.LISTING1, 1 << 20, "aos", "aos_aligned")
    assert "#define LLB_NS 2u" in s and "#define LLB_T 512u" in s and "#define LLB_G 4u" in s
    s = src(W.LISTING1, 1 << 20, "aos_aligned", "aosoa32")
    assert "#define LLB_NS 2u" in s and "#define LLB_T 256u" in s
    assert "#define LLB_NS 3u" in src(W.HEP100, 1 << 16, "aos", "aosoa32")  # (wide records: the rule stays off)
    assert "#define LLB_NS 4u" in src(W.HEP100, 1 << 16, "aos", "soa_mb")
    assert "#define LLB_NS 3u" in src(W.HEP100, 1 << 16, "aos_aligned", "soa_mb")
    assert "#define LLB_NS 3u" in src(W.HEP100, 1 << 16, "aos", "soa_mb", knobs={"jit_stages": 3})
    # record groups into SoA MB: no staging image for the destination leaves
    s0 = src(W.LISTING1, 1 << 20, "aos", "soa_mb")
    s2 = src(W.LISTING1, 1 << 20, "aos", "soa_mb", knobs={"jit_soa_tma": 2})
    assert s0 != s2
