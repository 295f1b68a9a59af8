"""Host-side logic of bench.py (CPU): the aggregation call widths per epoch (reading Q7), SURVEY
§8(d) d.4's SpMM fractions, and the config keys both arms report."""
import argparse
import types

import pytest

import bench
from paper_2512_01678_b200 import pad_width


def _fake_model(dims, order):
    return types.SimpleNamespace(dims=dims, order=order)


P = types.SimpleNamespace(pad_width=pad_width)


@pytest.mark.parametrize("dims,order,want", [
    ((602, 128, 41), [0, 0], [128, 48, 48, 128]),                 # reddit: two transform-first layers
    ((100, 256, 256, 47), [1, 0, 0], [104, 256, 48, 48, 256]),    # products: aggregate-first layer 1
    ((128, 256, 256, 40), [1, 0, 0], [128, 256, 40, 40, 256]),    # arxiv
])
def test_spmm_widths(dims, order, want):
    assert bench._spmm_widths(P, _fake_model(dims, order)) == want


def test_spmm_fractions_floor():
    # one 64-wide call on a graph whose operand fits L2: the floor is the L2-gather time
    r = {"kernels": {"spmm": {"ms_per_epoch": 2.0, "avg_launch_ms": 2.0, "algorithmic_GBps": 10000.0}},
         "_spmm_geometry": {"widths": [64], "n_rows": 1000, "n_cols": 1000, "nnz": 10 ** 8},
         "roofline": {"traffic": 1.0e9}}
    fr = bench._spmm_fractions(r, peak_hbm=8000.0, l2_gather_gbps=16000.0, l2_bytes=126 << 20)
    t_l2 = 1e8 * 4 * 64 / 16000e6          # ms
    assert fr["floor_ms_per_epoch"] == pytest.approx(t_l2)
    assert fr["time_efficiency_E"] == pytest.approx(t_l2 / 2.0)
    assert fr["dram_frac_of_hbm"] == pytest.approx(1.0e9 / 2.0e6 / 8000.0)
    assert fr["effective_frac_of_hbm"] == pytest.approx(10000.0 / 8000.0)
    # operand larger than L2: the HBM floor (each row once) applies
    r["_spmm_geometry"]["n_cols"] = r["_spmm_geometry"]["n_rows"] = 10 ** 7
    fr = bench._spmm_fractions(r, peak_hbm=8000.0, l2_gather_gbps=16000.0, l2_bytes=126 << 20)
    floor = 4.0 * 64 * 2e7 + 4.0 * 1e8 + 8.0 * (1e7 + 1) + 4.0 * 1e7
    assert fr["floor_ms_per_epoch"] == pytest.approx(floor / 8000e6)


def test_config_keys_shared_by_both_arms():
    a = argparse.Namespace(config="reddit", partition="1d", comm="p2p", gpus=1)
    one = bench._config_common(a, 1)
    assert one["workload"] == "reddit" and one["nodes"] == 232965 and one["parallelism"] == "single-gpu"
    four = bench._config_common(a, 4)
    assert four["parallelism"] == "1d-row-partition x4, comm p2p"
    assert set(one) == set(four)


def test_roofline_bounds(tmp_path, monkeypatch):
    """The aggregation's gathered (algorithmic, no-reuse) bytes are measured against the L2
    delivery ceiling of this run (max of the probes); GEMM-dominated epochs against HBM."""
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    peaks = {"hbm_gbs": 6500.0, "hbm_kind": "measured", "l2_stream_GBps": 21000.0,
             "gather": {"l2_resident_64MB": 16000.0, "hbm_resident_4GB": 5000.0}}
    k = {"spmm": {"ms_per_epoch": 8.0, "avg_launch_ms": 2.0, "algorithmic_GBps": 19000.0, "bytes_per_launch": 3.8e10},
         "gemm_nt": {"ms_per_epoch": 0.5, "avg_launch_ms": 0.1, "algorithmic_GBps": 5000.0, "bytes_per_launch": 5e8}}
    r = bench._roofline(k, 9.0, "reddit", peaks)
    assert r["bound"] == "l2" and r["kernel"] == "spmm" and r["peak"] == 21000.0   # no ncu peak: probes
    assert r["frac"] == pytest.approx(19000.0 / 21000.0)
    assert r["traffic"] is None and "dram_frac_of_hbm" not in r
    (tmp_path / "profiles").mkdir()
    (tmp_path / "profiles" / "l2_peak.json").write_text('{"lts_bytes_peak_GBps": 34650.0}')
    r = bench._roofline(k, 9.0, "reddit", peaks)
    assert r["peak"] == 34650.0 and r["frac"] == pytest.approx(19000.0 / 34650.0) and "ncu" in r["peak_source"]
    (tmp_path / "profiles" / "ncu_traffic_reddit.json").write_text('{"spmm": {"dram_bytes_per_launch": 1.0e9}}')
    r = bench._roofline(k, 9.0, "reddit", peaks)
    assert r["dram_frac_of_hbm"] == pytest.approx(1.0e9 / 2.0e6 / 6500.0)
    k2 = {"gemm_nt": k["gemm_nt"], "spmm": dict(k["spmm"], ms_per_epoch=0.1)}
    r = bench._roofline(k2, 1.0, "arxiv", peaks)
    assert r["bound"] == "hbm" and r["peak"] == 6500.0 and r["frac"] == pytest.approx(5000.0 / 6500.0)
