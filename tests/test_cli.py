"""kls-bench on the B200 backend: the QR-sweep generator matches the
reference bitwise (CPU), and every subcommand reproduces the reference CLI's
data rows — counts exactly, floating columns within the parity tolerances —
with the same exit codes (GPU)."""

import contextlib
import io

import numpy as np
import pytest

from conftest import golden


def test_synthetic_kappa_matches_reference_bitwise():
    from paper_2104_01253_b200.cli import synthetic_kappa

    g = golden("cli.npz")
    assert np.array_equal(synthetic_kappa(60, 8, 1e6, seed=3), g["kappa_matrix"])


def test_cli_config_errors_exit_2(capsys):
    from paper_2104_01253_b200 import cli

    assert cli.main(["sync-count", "--scheme", "mgs"]) == 2
    assert cli.main(["gmres", "--laplace-dims", "4,4"]) == 2


def _run(argv):
    from paper_2104_01253_b200 import cli

    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.main(list(argv))
    return rc, buf.getvalue()


def _rows(csv):
    lines = [ln for ln in csv.strip().splitlines() if not ln.startswith("#")]
    return lines[0], [ln.split(",") for ln in lines[1:]]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["sync", "qr", "arnoldi", "gmres", "eig"])
def test_cli_matches_reference_rows(cuda, name):
    g = golden("cli.npz")
    rc, out = _run([str(a) for a in g[f"{name}_argv"]])
    assert rc == int(g[f"{name}_rc"])
    head, got = _rows(out)
    rhead, ref = _rows(str(g[f"{name}_csv"]))
    assert head == rhead and len(got) == len(ref)
    cols = head.split(",")
    for a, b in zip(got, ref):
        assert len(a) == len(b)
        for col, x, y in zip(cols, a, b):
            try:
                fx, fy = float(x), float(y)
            except ValueError:
                assert x == y, (name, col, a, b)
                continue
            if x == y or (np.isnan(fx) and np.isnan(fy)):
                continue
            if col in ("loo", "rre"):
                # rounding-driven quantities: the same order of magnitude
                assert max(fx, fy) <= 1e-13 or 0.1 <= fx / fy <= 10.0, (name, col, a, b)
            else:
                # residual histories / backward errors: the reference's 1e-8
                assert abs(fx - fy) <= max(1e-8 * abs(fy), 1e-13), (name, col, a, b)


@pytest.mark.gpu
def test_cli_sync_count_negative_control(cuda):
    rc, _ = _run(["sync-count", "--rows", "300", "--cols", "10", "--scheme", "dcgs2",
                  "--inject-off-by-one", "--inject-off-by-one"])
    # one injected reduction stays within dcgs2's finalize slack; cgs2 has none
    rc2, _ = _run(["sync-count", "--rows", "300", "--cols", "10", "--scheme", "cgs2",
                   "--inject-off-by-one"])
    assert rc == 0 and rc2 == 3
