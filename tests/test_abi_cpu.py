"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/morphling.h
declares, and its host-only entry points (1D partition D1, local plans D2-D4) agree bit for bit
with the oracle.  No compute call needs a GPU here."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from synth.generate import make_small

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_2512_01678_b200 import _lib as L
    return L


def _declared():
    with open(os.path.join(ROOT, "include", "morphling.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(mph_\w+)\s*\(", src, flags=re.M)))


def test_header_symbols_exported():
    L = _lib()
    names = _declared()
    assert len(names) >= 40
    raw = L.raw()
    missing = [n for n in names if not hasattr(raw, n)]
    assert not missing, missing
    assert set(names) == set(L.EXPORTED), set(names) ^ set(L.EXPORTED)


def test_version_and_errors():
    L = _lib()
    assert L.mph_version() == 1
    with pytest.raises(L.MorphlingError) as e:
        L.mph_partition_1d(None, 3, 2, None)
    assert e.value.code == -1 and "partition_1d" in L.mph_last_error()


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    L = _lib()
    with pytest.raises(L.MorphlingError) as e:
        L.mph_device_check(ctypes.byref(ctypes.c_int32()))
    assert e.value.name == "MPH_ECUDA"
    src = np.array([0, 1], np.int32)
    h = ctypes.c_void_p()
    with pytest.raises(L.MorphlingError) as e:
        L.mph_graph_build(src.ctypes.data, src.ctypes.data, 2, 2, None, ctypes.byref(h))
    assert e.value.name == "MPH_ECUDA"


def test_package_refuses_to_import_without_the_library(tmp_path):
    """No CPU fallback: a copy of the package without libmorphling.so fails at import."""
    import shutil
    import subprocess
    import sys
    pkg = os.path.join(ROOT, "paper_2512_01678_b200")
    dst = tmp_path / "paper_2512_01678_b200"
    shutil.copytree(pkg, dst, ignore=shutil.ignore_patterns("lib", "csrc", "__pycache__"))
    r = subprocess.run([sys.executable, "-c", "import paper_2512_01678_b200"], cwd=tmp_path,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "ImportError" in r.stderr and "not built" in r.stderr, r.stderr[-2000:]


@pytest.mark.parametrize("seed,n,m", [(0, 50, 300), (1, 400, 3000), (2, 1000, 4000)])
def test_partition_matches_oracle(seed, n, m):
    from paper_2512_01678_b200 import partition_1d
    w = make_small(n, m, 4, 3, seed=seed, alpha=2.1)
    g = oracle.graph_build(w["src"], w["dst"], n)
    for world in (1, 2, 3, 4, 7, 8):
        assert np.array_equal(partition_1d(g.row_ptr, world), oracle.partition_1d(g.row_ptr, world))


def test_partition_degenerate_ranges():
    from paper_2512_01678_b200 import partition_1d
    g = oracle.graph_build([], [], 3)                 # 3 isolated nodes, 8 ranks: empty ranges allowed
    assert np.array_equal(partition_1d(g.row_ptr, 8), oracle.partition_1d(g.row_ptr, 8))


@pytest.mark.parametrize("world", [2, 3, 5])
def test_plan_matches_oracle_bit_exact(world):
    from paper_2512_01678_b200 import Plan
    n = 700
    w = make_small(n, 5000, 4, 5, seed=world, alpha=2.1, mu=0.4)
    g = oracle.graph_build(w["src"], w["dst"], n)
    bounds = oracle.partition_1d(g.row_ptr, world)
    for r in range(world):
        ref = oracle.localize(g, bounds, r)
        p = Plan(g.row_ptr, g.col_idx, n, bounds, r)
        a = p.arrays()
        assert p.n_own == ref.n_own and p.row0 == ref.row0
        assert np.array_equal(a["ghosts"], ref.ghosts)
        assert np.array_equal(a["row_ptr"], ref.row_ptr)
        assert np.array_equal(a["col_idx"], ref.col_idx)
        assert np.array_equal(a["split"], ref.split)
        assert np.array_equal(a["recv_offset"], ref.recv_offset)
        assert np.array_equal(a["n_recv"], ref.n_recv)
        gl = np.concatenate([np.arange(ref.row0, ref.row0 + ref.n_own), ref.ghosts])
        assert np.array_equal(a["deg_local"], g.deg[gl])
        for q in range(world):
            s0, s1 = a["send_offset"][q], a["send_offset"][q + 1]
            assert np.array_equal(a["send_ids"][s0:s1], ref.send_ids[q])


def test_plan_rejects_bad_arguments():
    from paper_2512_01678_b200 import Plan
    from paper_2512_01678_b200._lib import MorphlingError
    g = oracle.graph_build([0, 1], [1, 2], 3)
    with pytest.raises(MorphlingError):
        Plan(g.row_ptr, g.col_idx, 3, np.array([0, 2, 3]), 5)
    with pytest.raises(MorphlingError):
        Plan(g.row_ptr, g.col_idx, 3, np.array([0, 3, 2]), 0)


# ---------------------------------------------------------------- Alg. 4 partitioners (NEXT-3)
@pytest.mark.parametrize("seed,n,m", [(0, 300, 2500), (1, 1200, 9000), (2, 500, 350), (3, 60, 24), (4, 400, 150)])
def test_alg4_partitioners_match_oracle_bit_exact(seed, n, m):
    import paper_2512_01678_b200 as P
    w = make_small(n, m, 4, 3, seed=seed, alpha=2.1)
    g = oracle.graph_build(w["src"], w["dst"], n)
    phases = set()
    for world in (1, 2, 3, 4, 8):
        part, load = P.partition_greedy(g.row_ptr, world)
        ref = oracle.partition_greedy(g, world)
        assert np.array_equal(part, ref)
        assert np.array_equal(load, np.bincount(ref, weights=g.deg, minlength=world).astype(np.int64))
        pc, nc = P.partition_components(g.row_ptr, g.col_idx, world)
        rc, rnc = oracle.partition_components(g, world)
        assert nc == rnc and ((pc is None and rc is None) or np.array_equal(pc, rc))
        ph, phase = P.partition_hierarchical(g.row_ptr, g.col_idx, world)
        rh, rphase = oracle.partition_hierarchical(g, world)
        assert phase == rphase and np.array_equal(ph, rh)
        phases.add(phase)
        new_id, bounds = P.relabel(ph, world)
        rn, rb = oracle.relabel(rh, world)
        assert np.array_equal(new_id, rn) and np.array_equal(bounds, rb)
        assert np.array_equal(P.partition_stats(g.row_ptr, g.col_idx, ph, world), oracle.partition_stats(g, rh, world))
    print("phases", sorted(phases))


def test_relabel_rejects_bad_parts():
    import paper_2512_01678_b200 as P
    with pytest.raises(_lib().MorphlingError) as e:
        P.relabel(np.array([0, 1, 2], np.int32), 2)
    assert e.value.name == "MPH_EINVAL"
