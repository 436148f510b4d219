"""Reference-compatible CLI: schema on CPU, runs on GPU."""

import io
import sys
from contextlib import redirect_stdout

import pytest

REF = "/root/reference/pkg/src"


def test_columns_match_reference_schema():
    from paper_0912_4506_b200.cli import COLUMNS, build_parser
    # R/bench.py:26-27
    assert COLUMNS == ("variant", "nx", "ny", "nz", "n", "t", "T", "dl", "du", "dt",
                       "sync", "storage", "sweeps", "seconds", "mlups", "verified")
    a = build_parser().parse_args(["bench", "--dims", "16x8x4", "-T", "3", "--variant", "pipeline",
                                   "--depth", "3"])
    assert a.dims == (16, 8, 4) and a.updates_per_thread == 3 and a.depth == 3


def test_report_format():
    from paper_0912_4506_b200.cli import BenchResult, report
    from paper_0912_4506_b200 import GridDims, PipelineConfig
    r = BenchResult("gpu-naive", GridDims(16, 16, 16), PipelineConfig(), 2, 0.5, 8192, "yes")
    csv = report([r]).splitlines()
    assert csv[0].startswith("variant,nx,ny,nz") and csv[1].startswith("gpu-naive,16,16,16")
    assert '"mlups": "0.016"' in report([r], "json")


def _need_reference():
    """The CLI verifies against the reference package (baseline/_ref); skip where it is absent."""
    from paper_0912_4506_b200.cli import ReferenceUnavailable, _import_reference, build_parser
    try:
        _import_reference(build_parser().parse_args(["verify"]))
    except ReferenceUnavailable:
        pytest.skip("reference package not installed (pip install --target baseline/_ref)")


@pytest.mark.gpu
def test_cli_bench_verify_dist_on_gpu():
    _need_reference()
    from paper_0912_4506_b200.cli import cli_main
    out = io.StringIO()
    with redirect_stdout(out):
        rc = cli_main(["bench", "--size", "24", "--variant", "naive", "--variant", "pipeline",
                       "-T", "2", "--team-size", "2", "--sweeps", "3", "--reps", "1"])
    assert rc == 0, out.getvalue()
    lines = out.getvalue().splitlines()
    assert lines[1].startswith("gpu-naive") and lines[1].endswith(",yes")
    assert lines[2].startswith("gpu-pipeline") and lines[2].endswith(",yes")
    out = io.StringIO()
    with redirect_stdout(out):
        assert cli_main(["verify", "--size", "20", "-T", "4", "--team-size", "1", "--sweeps", "2",
                         "--depth", "3"]) == 0
        assert cli_main(["dist", "--dims", "12x10x32", "--layout", "1x1x2", "-T", "2",
                         "--team-size", "2", "--outer-steps", "2"]) == 0
    # the device is checked against the reference package's own code (baseline/_ref), never itself
    assert "/reference " in out.getvalue() and "(reference)" in out.getvalue()
    assert out.getvalue().count("PASS (bitwise") == 2


@pytest.mark.gpu
def test_cli_compressed_and_float32_on_gpu():
    """--storage compressed (R/bench.py:114,147-150,199-201; reference test_bench.py:81-92)
    and --dtype float32, both verified against the reference package."""
    _need_reference()
    from paper_0912_4506_b200.cli import cli_main
    out = io.StringIO()
    with redirect_stdout(out):
        rc = cli_main(["bench", "--size", "16", "--variant", "pipeline", "--storage", "compressed",
                       "--teams", "1", "--team-size", "2", "-T", "1", "--block", "16x8x8",
                       "--sweeps", "3", "--reps", "1"])
    assert rc == 0, out.getvalue()
    row = out.getvalue().strip().split("\n")[1].split(",")
    assert row[0] == "gpu-pipeline" and row[11] == "compressed" and row[-1] == "yes"
    out = io.StringIO()
    with redirect_stdout(out):
        assert cli_main(["verify", "--size", "16", "--storage", "compressed", "--team-size", "2",
                         "-T", "2", "--sweeps", "3"]) == 0
        assert cli_main(["verify", "--size", "20", "--dtype", "float32", "-T", "4", "--team-size", "1",
                         "--sweeps", "2"]) == 0
        assert cli_main(["dist", "--dims", "12x10x32", "--layout", "1x1x2", "-T", "2", "--team-size", "2",
                         "--outer-steps", "2", "--dtype", "float32"]) == 0
    assert "gpu-compressed/reference" in out.getvalue()


def test_reference_field_is_the_reference_code(O):
    """The CLI's verification field comes from the reference package's own sweep
    (baseline/_ref or --reference-path), bit-equal to the pinned oracle, fp32 included."""
    import os
    import numpy as np
    from paper_0912_4506_b200 import GridDims
    from paper_0912_4506_b200.cli import ReferenceUnavailable, _reference_field, build_parser
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if not os.path.isdir(os.path.join(root, "baseline", "_ref", "stencilpipe")) and not os.path.isdir(REF):
        pytest.skip("reference package not installed")
    a = build_parser().parse_args(["verify", "--size", "9", "--pattern", "random", "--seed", "7"] +
                                  ([] if os.path.isdir(os.path.join(root, "baseline", "_ref")) else
                                   ["--reference-path", REF]))
    d = GridDims(9, 8, 7)
    ref64, src = _reference_field(a, d, None, 3, np.float64)
    assert src == "reference"
    g = O.CGrid(d.shape, O.BoxPattern("random", seed=7))
    g.sweeps(3)
    assert np.array_equal(ref64.view(np.uint64), g.interior().view(np.uint64))
    ref32, _ = _reference_field(a, d, None, 3, np.float32)
    g32 = O.CGrid(d.shape, O.BoxPattern("random", seed=7), dtype=np.float32)
    g32.sweeps(3)
    assert ref32.dtype == np.float32 and np.array_equal(ref32.view(np.uint32), g32.interior().view(np.uint32))
    with pytest.raises(ReferenceUnavailable):
        _import_reference_no_default(build_parser().parse_args(["verify"]))


def _import_reference_no_default(args):
    import builtins
    real = builtins.__import__

    def fake(name, *a, **k):
        if name.startswith("stencilpipe"):
            raise ImportError(name)
        return real(name, *a, **k)
    builtins.__import__ = fake
    try:
        from paper_0912_4506_b200.cli import _import_reference
        _import_reference(args)
    finally:
        builtins.__import__ = real


@pytest.mark.gpu
def test_cli_dump_matches_oracle(O, tmp_path):
    """`bench --dump` (R/bench.py:187-189): the field a GPU run leaves -- the
    compressed pipeline included -- equals the oracle's, independent of the
    reference package (checked here by the test, not by the CLI)."""
    import numpy as np
    from paper_0912_4506_b200 import load_field
    from paper_0912_4506_b200.cli import cli_main
    for storage in ("twogrid", "compressed"):
        path = tmp_path / f"field_{storage}.txt"
        with redirect_stdout(io.StringIO()):
            assert cli_main(["bench", "--size", "16", "--variant", "pipeline", "--storage", storage,
                             "--teams", "1", "--team-size", "2", "-T", "2", "--sweeps", "3", "--reps", "1",
                             "--no-verify", "--dump", str(path)]) == 0
        with open(path) as fh:
            dims, field = load_field(fh)
        levels = (3 + 1) * 4                          # warm-up sweep + 3 timed, U = 4 each
        g = O.CGrid((16, 16, 16), O.BoxPattern("random", seed=42))
        g.sweeps(levels)
        assert np.array_equal(field[1:-1, 1:-1, 1:-1].view(np.uint64), g.interior().view(np.uint64)), storage
