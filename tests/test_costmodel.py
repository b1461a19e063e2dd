"""The cost model mirror against the reference's closed forms and the roofline
numbers DESIGN.md / SURVEY 8d quote."""

import math

import pytest

from paper_1507_00921_b200 import costmodel as cm


def test_reference_closed_forms():
    # costmodel.py:1-20: FFE N (8 log2 N + 8) / (N - M) mults; ESSFM N (8 log2 N + 21 + Nc) ...
    r = cm.cost_per_sample("ffe", 2048, 700)
    assert r.mults_per_sample == pytest.approx(2048 * (8 * 11 + 8) / 1348)
    assert r.adds_per_sample == pytest.approx(2048 * (8 * 11 + 4) / 1348)
    assert r.latency_proxy == 1 and r.num_steps == 1
    r = cm.cost_per_sample("essfm", 2048, 700, n_coeffs=17, num_steps=2)
    assert r.mults_per_sample == pytest.approx(2 * 2048 * (88 + 21 + 17) / 1348)
    assert r.adds_per_sample == pytest.approx(2 * 2048 * (88 + 11 + 34) / 1348)
    assert r.latency_proxy == 2 and r.power_proxy == r.mults_per_sample
    r = cm.cost_per_sample("ssfm", 1024, 256, n_coeffs=9, num_steps=20)
    assert r.n_coeffs == 0 and r.mults_rounded == round(20 * 1024 * (80 + 21) / 768)


@pytest.mark.parametrize("args", [("bogus", 2048, 700), ("ffe", 2000, 700), ("ffe", 2048, 2048),
                                  ("ffe", 2048, -1)])
def test_reference_errors(args):
    with pytest.raises(ValueError):
        cm.cost_per_sample(*args)
    with pytest.raises(ValueError):
        cm.cost_per_sample("essfm", 2048, 700, n_coeffs=-1)
    with pytest.raises(ValueError):
        cm.cost_per_sample("essfm", 2048, 700, num_steps=0)


def test_optimize_sweep_and_csv():
    n, rep = cm.optimize_block_length("essfm", 700, n_coeffs=17, candidates=[1024, 2048, 4096, 8192])
    best = min((cm.cost_per_sample("essfm", c, 700, 17).mults_per_sample, c) for c in (1024, 2048, 4096, 8192))
    assert (rep.mults_per_sample, n) == best
    with pytest.raises(ValueError):
        cm.optimize_block_length("ffe", 700, candidates=[512, 1024])
    with pytest.raises(ValueError):
        cm.optimize_block_length("ffe", 700, candidates=[])
    rows = cm.sweep_link_length(["ffe", "essfm"], [800.0, 3200.0], 21.68, 28e9, n_coeffs=9)
    assert [r.algorithm for r in rows] == ["ffe", "essfm", "ffe", "essfm"]
    assert all(r.block_len == 8 * r.overlap for r in rows)
    csv = cm.cost_table_csv(rows)
    lines = csv.strip().split("\n")
    assert lines[0].startswith("algorithm,N,M,Nc,Ns") and len(lines) == 5
    assert max(float(l.split(",")[-1]) for l in lines[1:]) == 100.0
    with pytest.raises(ValueError):
        cm.cost_table_csv([])


def test_b200_roofline_matches_survey_table():
    # configs[0] symmetric 814.3 flop / 40.31 B, FP32-bound 91.4 GS/s
    r = cm.b200_roofline("essfm", 2048, 700, n_coeffs=17, num_steps=1)
    assert r.flops_per_sample == pytest.approx(814.338, abs=1e-2)
    assert r.bytes_per_sample == pytest.approx(40.3086, abs=1e-3)
    assert r.bound == "fp32" and r.roofline_gsps == pytest.approx(91.4, abs=0.3)
    # linear-first 461.9 flop; SSFM-20 linear-first 7687.6 flop
    assert cm.b200_roofline("essfm", 2048, 700, 17, 1, "linear-first").flops_per_sample == pytest.approx(461.9, abs=0.1)
    assert cm.b200_roofline("ssfm", 2048, 700, 0, 20, "linear-first").flops_per_sample == pytest.approx(7687.6, abs=0.1)
    # FFE 4096/700: HBM-bound at the measured bandwidth
    f = cm.b200_roofline("ffe", 4096, 700)
    assert f.bound == "hbm" and f.roofline_gsps == pytest.approx(6548.2 / f.bytes_per_sample, rel=1e-9)
    assert f.intensity == pytest.approx(f.flops_per_sample / f.bytes_per_sample)
    n, best = cm.optimize_block_length_b200("ffe", 700)
    assert best.roofline_gsps == max(cm.b200_roofline("ffe", c, 700).roofline_gsps for c in (1024, 2048, 4096, 8192))
    assert math.isclose(cm.B200_FP32_TFLOPS, 74.4, rel_tol=1e-3)


def test_matches_the_reference_cost_model_when_installed():
    # the unmodified reference in oracle/_ref (oracle/install_ref.sh), when present
    import importlib
    import sys
    from pathlib import Path

    ref = Path(__file__).resolve().parent.parent / "oracle" / "_ref"
    if not (ref / "fiberdbp" / "costmodel.py").exists():
        pytest.skip("reference not installed in oracle/_ref")
    sys.path.insert(0, str(ref))
    try:
        rcm = importlib.import_module("fiberdbp.costmodel")
    except Exception as e:   # numba & co. missing on this host
        pytest.skip(f"reference not importable: {e}")
    finally:
        sys.path.remove(str(ref))
    for alg in ("ffe", "ssfm", "essfm"):
        for n, m in ((256, 64), (2048, 700), (8192, 1024)):
            for nc, ns in ((0, 1), (17, 1), (33, 4)):
                a, b = cm.cost_per_sample(alg, n, m, nc, ns), rcm.cost_per_sample(alg, n, m, nc, ns)
                assert (a.mults_per_sample, a.adds_per_sample, a.latency_proxy, a.n_coeffs, a.num_steps) == \
                       (b.mults_per_sample, b.adds_per_sample, b.latency_proxy, b.n_coeffs, b.num_steps)
    rows = cm.sweep_link_length(["ffe", "ssfm", "essfm"], [80.0, 1600.0, 3200.0], 21.68, 56e9, 9)
    rrows = rcm.sweep_link_length(["ffe", "ssfm", "essfm"], [80.0, 1600.0, 3200.0], 21.68, 56e9, 9)
    assert cm.cost_table_csv(rows) == rcm.cost_table_csv(rrows)
    assert cm.optimize_block_length("essfm", 700, 17, [1024, 2048, 4096])[0] == \
           rcm.optimize_block_length("essfm", 700, 17, [1024, 2048, 4096])[0]
