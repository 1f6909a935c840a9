"""sim_study + cli.

CPU: the oracle's Gauss-Legendre restatement of Eq. 19-20 pinned against the
reference's own quadrature (oracle/_ref), the SPEC's est_bias / est_mse
examples, the seed mixing, and the CLI's data/usage errors.
GPU: pcb_rel_error against the oracle, run_study's M = 1 identities and
reproducibility, split-fit M = 1 == fit.
"""

import pytest

import paper_1609_05530_b200 as pcb
from paper_1609_05530_b200 import cli
from paper_1609_05530_b200.study import ReplicateRow, est_bias, est_mse, mix_seed

CASES = [(0, 0.3, 0.31), (0, -0.7, -0.65), (1, 5.0, 5.2), (1, -5.0, -4.0), (2, 2.0, 2.1), (2, 1.0, 1.05)]


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


@pytest.mark.parametrize("fam,ta,tb", CASES)
def test_oracle_rel_error_matches_reference(orc, ref, fam, ta, tb):
    if ref is None:
        pytest.skip("oracle/_ref not built")
    a, b = orc.rel_error(fam, ta, tb, 64), ref.rel_error(fam, ta, tb, 64)
    assert rel(a[0], b[0]) <= 1e-12 and rel(a[1], b[1]) <= 1e-12


def test_oracle_rel_error_identities(orc):
    for fam, ta, _ in CASES:
        assert orc.rel_error(fam, ta, ta, 64) == (0.0, 0.0)
    # continuity: -> 0 as theta_b -> theta_a
    vals = [orc.rel_error(2, 2.0, 2.0 + d, 64)[0] for d in (1e-1, 1e-2, 1e-3)]
    assert vals[0] > vals[1] > vals[2] > 0.0


def test_est_bias_mse_spec_examples():
    rows = [ReplicateRow(0, 0, 0.2, 0.3, 0, 0), ReplicateRow(1, 0, 0.5, 0.5, 0, 0)]
    assert est_mse(rows) == pytest.approx(0.005, rel=1e-15)
    same = [ReplicateRow(0, 0, 0.3, 0.3, 0, 0)] * 3
    assert est_bias(same) == 0.0 and est_mse(same) == 0.0
    assert est_bias([ReplicateRow(0, 0, 0.30, 0.31, 0, 0)]) == pytest.approx(0.01, rel=1e-12)


def test_mix_seed_matches_oracle(orc):  # rng.hpp:24-29
    fn = orc.lib.orc_mix_seed4
    for base, w in [(1, (2, 3, 4, 5)), (0x160905530, (0, 50000, 10, 7)), (2**64 - 1, (2, 2**63, 1, 0))]:
        assert mix_seed(base, w) == fn(base, *w)


def test_cli_data_and_usage_errors(tmp_path):
    one = tmp_path / "one.csv"
    one.write_text("x\n" + "\n".join(str(i) for i in range(40)) + "\n")
    assert cli.main(["fit", str(one)]) == 3  # "expected 2 numeric columns"
    bad = tmp_path / "bad.csv"
    bad.write_text("a,b\n" + "\n".join(f"{i},z" for i in range(40)) + "\n")
    assert cli.main(["fit", str(bad)]) == 3
    short = tmp_path / "short.csv"
    short.write_text("\n".join(f"{i},{i}" for i in range(5)) + "\n")
    assert cli.main(["fit", str(short)]) == 3
    assert cli.main(["fit", str(one), "--family", "clayton"]) == 2
    assert cli.main(["nope"]) == 2
    c1, c2 = cli.read_csv(str(_write_pairs(tmp_path / "h.csv", header=True)))
    assert len(c1) == 100 and c2[3] == 0.5 * 3


def _summary(path, rows):
    path.parent.mkdir(parents=True, exist_ok=True)
    head = ",".join(cli.SUMMARY_COLS)
    path.write_text(cli.SCHEMA + "\n" + head + "\n" + "\n".join(",".join(str(x) for x in r) for r in rows) + "\n")


def test_cli_report(tmp_path, capsys):
    empty = tmp_path / "empty"
    empty.mkdir()
    assert cli.main(["report", str(empty)]) == 3  # "no results found"
    res = tmp_path / "results"
    _summary(res / "g" / "summary.csv", [[0, 0.3, 50000, 10, 5, 0.3, 0.301, 0.001, 2e-6, 0.01, 0.012, 0.5, 20.0, 1],
                                         [0, 0.3, 50000, 100, 5, 0.3, 0.302, 0.002, 5e-6, 0.02, 0.03, 0.05, 21.0, 1]])
    _summary(res / "f" / "summary.csv", [[1, 5.0, 50000, 10, 5, 5.0, 5.01, 0.01, 1e-4, 0.01, 0.02, 0.7, 30.0, 2]])
    bad = res / "old" / "summary.csv"
    bad.parent.mkdir(parents=True)
    bad.write_text("# parcop-b200 csv schema v0\nfamily\n")
    assert cli.main(["report", str(res), "--out", str(tmp_path / "rep")]) == 0
    err = capsys.readouterr().err
    assert "schema mismatch" in err
    timing = (tmp_path / "rep" / "report_timing.csv").read_text().splitlines()
    assert timing[0] == cli.SCHEMA and timing[1] == "family,N,subset_s_M10,subset_s_M100,full_s"
    assert timing[2] == "gaussian,50000,0.5,0.05,20.5" and timing[3] == "frank,50000,0.7,,30.0"
    acc = (tmp_path / "rep" / "report_accuracy.csv").read_text().splitlines()
    assert len(acc) == 2 + 3 and acc[2].startswith("gaussian,0.3,50000,10,5,0.001,")


def _write_pairs(path, header):
    lines = (["u,v"] if header else []) + [f"{i * 0.01!r},{0.5 * i!r}" for i in range(100)]
    path.write_text("\n".join(lines) + "\n")
    return path


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("fam,ta,tb", CASES)
def test_device_rel_error_parity(ctx, orc, fam, ta, tb):
    for nodes in (64, 200):
        d = pcb.rel_error(fam, ta, tb, nodes, ctx=ctx)
        o = orc.rel_error(fam, ta, tb, nodes)
        assert rel(d[0], o[0]) <= 1e-9 and rel(d[1], o[1]) <= 1e-9
    assert pcb.rel_error(fam, ta, ta, 200, ctx=ctx) == (0.0, 0.0)


@pytest.mark.gpu
def test_device_rel_error_errors(ctx):
    with pytest.raises(pcb.DomainError):
        pcb.rel_error(2, 0.5, 2.0, 64, ctx=ctx)
    with pytest.raises(ValueError):
        pcb.rel_error(0, 0.1, 0.2, 0, ctx=ctx)


@pytest.mark.gpu
def test_run_study_m1_identities_and_reproducibility(ctx):
    cfg = pcb.SimConfig(0, 0.3, 20000, 1, S=2, quad_nodes=64)
    r = pcb.run_study(cfg, ctx=ctx)
    assert r.bias_hat == 0.0 and r.mse_hat == 0.0 and r.rel_l1 == 0.0 and r.rel_l2 == 0.0
    cfg = pcb.SimConfig(2, 2.0, 20000, 10, S=2, quad_nodes=64)
    a, b = pcb.run_study(cfg, ctx=ctx), pcb.run_study(cfg, ctx=ctx)
    assert [(x.theta_full, x.theta_combined) for x in a.per_replicate] == \
        [(x.theta_full, x.theta_combined) for x in b.per_replicate]
    assert a.mse_hat >= (sum(x.theta_combined - x.theta_full for x in a.per_replicate) / 2) ** 2 - 1e-18
    assert a.rel_l1 > 0.0 and abs(a.bias_hat) < 0.05


@pytest.mark.gpu
def test_cli_split_fit_m1_equals_fit(ctx, tmp_path, capsys):
    X = pcb.sample_matrix(1, 5.0, 5000, 1, ctx=ctx)
    p = tmp_path / "x.csv"
    p.write_text("\n".join(f"{float(a)!r},{float(b)!r}" for a, b in zip(X.col1, X.col2)) + "\n")
    assert cli.main(["fit", str(p), "--family", "frank"]) == 0
    fit_line = capsys.readouterr().out.strip().splitlines()[-1]
    out = tmp_path / "blocks.csv"
    assert cli.main(["split-fit", str(p), "--family", "frank", "--subsets", "1", "--out", str(out)]) == 0
    comb_line = capsys.readouterr().out.strip().splitlines()[-1]
    th_fit = float(fit_line.split()[0].split("=")[1])
    th_comb = float(comb_line.split()[0].split("=")[1])
    assert th_fit == th_comb
    assert out.read_text().startswith(cli.SCHEMA)
