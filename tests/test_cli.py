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


@pytest.mark.gpu
def test_cli_bench_verify_dist_on_gpu():
    from paper_0912_4506_b200.cli import cli_main
    out = io.StringIO()
    with redirect_stdout(out):
        rc = cli_main(["bench", "--size", "24", "--variant", "naive", "--variant", "pipeline",
                       "-T", "2", "--team-size", "2", "--sweeps", "3", "--reps", "1"])
    assert rc == 0, out.getvalue()
    lines = out.getvalue().splitlines()
    assert lines[1].startswith("gpu-naive") and lines[1].endswith(",yes")
    assert lines[2].startswith("gpu-pipeline") and lines[2].endswith(",yes")
    with redirect_stdout(io.StringIO()):
        assert cli_main(["verify", "--size", "20", "-T", "4", "--team-size", "1", "--sweeps", "2",
                         "--depth", "3"]) == 0
        assert cli_main(["dist", "--dims", "12x10x32", "--layout", "1x1x2", "-T", "2",
                         "--team-size", "2", "--outer-steps", "2"]) == 0
