"""The experiment CLI and batch builders on the GPU solve vs the reference's
own CLI output (tests/golden/cli, made by running batchode.cli in
tests/golden/make_golden.py cli): identical CSV schemas, instance rows,
step counts and statuses; traces and the limit cycle within tolerance."""
import csv
import os

import numpy as np
import pytest

from paper_2210_12375_b200 import cli, problems

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")
RUNS = {
    "vdp_ind": ["vdp-batching", "--n", "4", "--mu", "25"],
    "vdp_joint": ["vdp-batching", "--n", "4", "--mu", "25", "--mode", "joint"],
    "vdp_random_tsit5_pi42": ["vdp-batching", "--n", "6", "--mu", "5", "--random-phases", "--seed",
                              "3", "--controller", "pid:PI42", "--method", "tsit5", "--n-eval", "0"],
    "pid_sweep": ["pid-sweep", "--mu", "5,25"],
}


def read(path):
    with open(path, newline="") as fh:
        rows = list(csv.reader(fh))
    return rows[0], rows[1:]


def test_limit_cycle_and_batch_match_reference():
    g = np.load(os.path.join(HERE, "problems.npz"))
    anchor, period = problems.vdp_limit_cycle(25.0)
    np.testing.assert_allclose(anchor, g["anchor"], rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(period, g["period"], rtol=1e-9)
    batch = problems.vdp_batch(4, 25.0, n_eval=5)
    np.testing.assert_allclose(batch.y0, g["y0"], rtol=1e-8, atol=1e-8)
    np.testing.assert_allclose(batch.t_end, g["t_end"], rtol=1e-9)
    np.testing.assert_allclose(np.array(batch.t_eval), g["t_eval"], rtol=1e-9)


@pytest.mark.parametrize("name", sorted(RUNS))
def test_cli_rows_match_reference(name, tmp_path):
    argv = RUNS[name] + ["--out", str(tmp_path / "rows.csv")]
    if argv[0] == "vdp-batching":
        argv += ["--trace-out", str(tmp_path / "trace.csv")]
    assert cli.main(argv) == 0
    h, rows = read(tmp_path / "rows.csv")
    gh, grows = read(os.path.join(HERE, name + ".csv"))
    assert h == gh and len(rows) == len(grows)
    # pid-sweep integrates one instance from the limit-cycle anchor that the
    # CLI itself computes (vdp_limit_cycle, agreeing with the reference to
    # ~1e-10): a step count next to an accept/reject boundary may move by a
    # step or two there, so its counts are compared at 1%
    loose = name == "pid_sweep"
    for r, g in zip(rows, grows):
        for col, a, b in zip(h, r, g):
            if col == "ratio_vs_integral":
                assert abs(float(a) - float(b)) <= (1e-2 if loose else 1e-9) * abs(float(b)), (col, a, b)
            elif loose and col in ("n_steps", "n_accepted"):
                assert abs(int(a) - int(b)) <= 0.01 * int(b), (col, a, b)
            else:
                assert a == b, (col, a, b)
    if argv[0] == "vdp-batching":
        th, trows = read(tmp_path / "trace.csv")
        gth, gtrows = read(os.path.join(HERE, name + "_trace.csv"))
        assert th == gth and len(trows) == len(gtrows)
        a = np.array([[float(x) for x in r] for r in trows])
        b = np.array([[float(x) for x in r] for r in gtrows])
        assert np.array_equal(a[:, :2], b[:, :2])             # instance, step
        np.testing.assert_allclose(a[:, 2], b[:, 2], rtol=1e-7, atol=1e-9)  # t
        np.testing.assert_allclose(a[:, 3], b[:, 3], rtol=1e-5)             # dt


def test_looptime_schema(tmp_path):
    out = tmp_path / "loop.csv"
    assert cli.main(["looptime", "--n", "4096", "--steps", "200", "--repeats", "2",
                     "--out", str(out)]) == 0
    h, rows = read(out)
    assert h == ["run", "n", "d", "steps", "loop_time_us"]
    assert [r[0] for r in rows] == ["1", "2", "mean+-sd"]
    assert all(int(r[3]) >= 200 for r in rows)
