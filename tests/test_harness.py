"""nbsim CLI / report / snapshot parity.

Goldens come from running the reference's own CLI (tests/golden/make_golden.py
gen_report): report_alg{0,1}.txt and snapshot_alg{0,1}_000004.csv."""

import os

import numpy as np
import pytest

from paper_2203_08966_b200 import harness
from paper_2203_08966_b200.physics import Bodies
from paper_2203_08966_b200.simulation import SimConfig

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _report(path):
    out = {}
    for line in open(path).read().splitlines():
        k, v = line.split(" = ", 1)
        out[k] = v
    return out


def test_snapshot_roundtrip_bit_exact(tmp_path):
    rng = np.random.default_rng(0)
    b = Bodies(rng.random(50), rng.normal(size=(50, 3)) * 1e3, rng.normal(size=(50, 3)) * 1e-7)
    p = tmp_path / "s.csv"
    harness.emit_snapshot(p, 0.30000000000000004, b)
    t, c = harness.read_snapshot(p)
    assert t == 0.30000000000000004
    np.testing.assert_array_equal(c.mass, b.mass)
    np.testing.assert_array_equal(c.position, b.position)
    np.testing.assert_array_equal(c.velocity, b.velocity)


@pytest.mark.parametrize("alg", [0, 1])
def test_reference_snapshot_reads_and_rewrites_identically(tmp_path, alg):
    src = os.path.join(GOLD, f"snapshot_alg{alg}_000004.csv")
    t, b = harness.read_snapshot(src)
    harness.emit_snapshot(tmp_path / "x.csv", t, b)
    assert (tmp_path / "x.csv").read_text() == open(src).read()


def test_snapshot_header_errors(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text("t=1 n=2\n")
    with pytest.raises(ValueError, match="not a snapshot"):
        harness.read_snapshot(p)
    p.write_text("# t=0.0 n=3\n1,2,3,4,5,6,7\n")
    with pytest.raises(ValueError, match="header says 3"):
        harness.read_snapshot(p)


@pytest.mark.parametrize("alg", [0, 1])
def test_report_schema_matches_reference(alg):
    """RunReport.lines() rebuilt from the golden's values reproduces every
    line of the reference report, in order (timing lines included)."""
    gold = open(os.path.join(GOLD, f"report_alg{alg}.txt")).read()
    g = _report(os.path.join(GOLD, f"report_alg{alg}.txt"))
    cfg = SimConfig(n=int(g["n"]), algorithm=int(g["algorithm"]), ranks=int(g["ranks"]),
                    theta=float(g["theta"]), dt=float(g["dt"]), steps=int(g["steps"]), eps=float(g["eps"]),
                    seed=int(g["seed"]))
    audits = []
    i = 0
    while f"audit_{i}_t" in g:
        audits.append((float(g[f"audit_{i}_t"]), float(g[f"audit_{i}_energy"])))
        i += 1
    phases = harness.PHASES
    per = {p: float(g[f"time_rank0_{p}"]) for p in phases}
    rep = harness.RunReport(config=cfg, transport=g["transport"], energy_initial=float(g["energy_initial"]),
                            energy_final=float(g["energy_final"]),
                            drift_percent=float(g["energy_drift_percent"]),
                            child_requests=int(g["child_requests"]),
                            message_totals={p: (int(g[f"msgs_{p}"]), int(g[f"bytes_{p}"])) for p in phases},
                            audits=audits, phase_seconds=[per], wall_seconds=float(g["wall_seconds"]))
    assert rep.to_text() == gold
    assert "time_" not in rep.deterministic_text() and "wall_" not in rep.deterministic_text()


def test_cli_argument_errors(capsys):
    with pytest.raises(SystemExit):
        harness.main(["--algorithm", "1", "--n", "100", "--snapshot-every", "2"])
    with pytest.raises(SystemExit):
        harness.main(["--algorithm", "1", "--n", "100", "--audit-every", "0"])
    with pytest.raises(SystemExit):
        harness.main(["--algorithm", "9", "--n", "100"])
    with pytest.raises(SystemExit):
        harness.main(["--algorithm", "1", "--n", "2"])  # SimConfig: need at least 4 bodies


def test_scaling_csv_columns():
    rows = [dict(algorithm=1, n=10, ranks=1, wall_time=1.0, speedup_vs_ranks1=1.0, parallel_cost=0.1, error="")]
    assert harness.scaling_csv(rows).splitlines() == [
        "algorithm,n,ranks,wall_time,speedup_vs_ranks1,parallel_cost,error", "1,10,1,1.0,1.0,0.1,"]


@pytest.mark.gpu
@pytest.mark.parametrize("alg,n,steps", [(1, 600, 8), (0, 300, 4)])
def test_cli_run_matches_reference_report(tmp_path, alg, n, steps):
    """The GPU run of the reference's CLI arguments (fp64): the same report
    lines; counts exact, energies and the snapshot within 1e-12 relative."""
    args = ["--algorithm", str(alg), "--n", str(n), "--steps", str(steps), "--dt", "0.01", "--eps", "0.05",
            "--seed", "3", "--snapshot-every", "4", "--audit-every", "4", "--out", str(tmp_path)]
    assert harness.main(args) == 0
    got = _report(tmp_path / "report.txt")
    gold = _report(os.path.join(GOLD, f"report_alg{alg}.txt"))
    assert list(got) == list(gold)
    for k, v in gold.items():
        if k.startswith(("time_", "wall_")):
            continue
        if k == "energy_drift_percent":
            continue
        if "energy" in k or k.endswith("_t") or k in ("theta", "dt", "eps"):
            assert float(got[k]) == pytest.approx(float(v), rel=1e-12, abs=1e-15), k
        else:
            assert got[k] == v, k
    # the drift itself: within 1% of the reference's
    d_got, d_ref = float(got["energy_drift_percent"]), float(gold["energy_drift_percent"])
    assert abs(d_got - d_ref) <= 0.01 * abs(d_ref) + 1e-12
    t, b = harness.read_snapshot(tmp_path / "snapshot_000004.csv")
    t0, b0 = harness.read_snapshot(os.path.join(GOLD, f"snapshot_alg{alg}_000004.csv"))
    assert t == t0
    np.testing.assert_array_equal(b.mass, b0.mass)
    np.testing.assert_allclose(b.position, b0.position, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(b.velocity, b0.velocity, rtol=1e-12, atol=1e-14)
