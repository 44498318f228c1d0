"""Model arithmetic (restating the reference's tests/test_perf.py model
checks), the GPU traffic model, and the CLI (host-side parts on CPU)."""

import json
from fractions import Fraction

import pytest

from paper_1004_1741_b200.cli import build_parser, main
from paper_1004_1741_b200.errors import DomainError
from paper_1004_1741_b200.perf import predict_p0, predict_traffic


def test_predict_p0_reference_values():
    assert predict_p0(18.5e9, 16) == 1.15625e9   # Nehalem EP
    assert predict_p0(4.8e9, 16) == 300e6
    assert predict_p0(6534.5e9, 16) == 408.40625e9  # B200 measured copy bandwidth


def test_predict_p0_domain():
    for ms, b in ((0, 16), (-1.0, 16), (16, 0), (16, -2)):
        with pytest.raises(DomainError):
            predict_p0(ms, b)


def test_traffic_identities():
    for t in range(1, 17):
        for kernel, nt in (("jacobi", True), ("jacobi", False), ("gs", None)):
            assert predict_traffic(kernel, "wavefront", t, nt) * t == predict_traffic(kernel, "plain", 1, nt)
        assert predict_traffic("jacobi", "wavefront", t, device="b200") == Fraction(16, t)
    assert predict_traffic("gs", "wavefront", 6) == Fraction(16, 6)
    assert predict_traffic("jacobi", "plain", 1, nt_stores=False) == 24
    assert predict_traffic("jacobi", "plain", 1, device="b200") == 16
    with pytest.raises(DomainError):
        predict_traffic("gs", "plain", 1, nt_stores=True)
    with pytest.raises(DomainError):
        predict_traffic("jacobi", "plain", 0)
    with pytest.raises(DomainError):
        predict_traffic("jacobi", "bogus", 1)


def test_cli_model(capsys):
    assert main(["model", "--ms", "6534.5e9", "--gpu", "--variant", "wavefront", "--tpg", "4"]) == 0
    rec = json.loads(capsys.readouterr().out)
    assert rec["bytes_per_lup"] == 4.0 and rec["p0_mlups"] == pytest.approx(1633625.0)


def test_cli_usage_errors_exit_2(capsys):
    assert main(["verify", "--kernel", "jacobi", "--variant", "wavefront", "--tpg", "3",
                 "--iters", "4"]) == 2
    with pytest.raises(SystemExit):
        build_parser().parse_args(["bench", "--size", "10x10"])


@pytest.mark.gpu
def test_cli_verify_and_bench(capsys, tmp_path):
    for kernel in ("jacobi", "gs-naive", "gs-interleaved"):
        assert main(["verify", "--kernel", kernel, "--variant", "wavefront", "--tpg", "2",
                     "--iters", "6", "--size", "30x22x18", "--a", "0.0"]) == 0
    assert main(["verify", "--kernel", "jacobi", "--variant", "serial", "--iters", "5",
                 "--size", "31x20x17", "--a", "0.5", "--b", "0.1"]) == 0
    out = tmp_path / "r.json"
    assert main(["bench", "--size", "64x64x64", "--iters", "8", "--tpg", "4", "--reps", "2",
                 "--format", "json", "--out", str(out), "--dump-grid", str(tmp_path / "g.bin")]) == 0
    rec = json.loads(out.read_text())
    assert rec["depth"] == 4 and rec["mlups"] > 0 and 0 < rec["hbm_frac"] < 5
    assert (tmp_path / "g.bin").stat().st_size == 24 + 64 ** 3 * 8


@pytest.mark.gpu
def test_cli_gpus_threaded_and_pipeline(capsys, tmp_path):
    """--devices / --gpus run the threaded engines as z-slabs over GPUs
    (one GPU here: slabs share it), checked bitwise against the serial
    engine like the reference's verify (cli.py:297-331)."""
    for kernel, variant in (("jacobi", "threaded"), ("gs-naive", "pipeline"),
                            ("gs-interleaved", "threaded")):
        assert main(["verify", "--kernel", kernel, "--variant", variant, "--iters", "7",
                     "--size", "30x22x18", "--devices", "0,0,0"]) == 0
    out = tmp_path / "r.json"
    assert main(["bench", "--kernel", "jacobi", "--variant", "threaded", "--size", "64x64x64",
                 "--iters", "8", "--reps", "2", "--devices", "0,0", "--format", "json",
                 "--out", str(out)]) == 0
    rec = json.loads(out.read_text())
    assert rec["gpus"] == 2 and rec["mlups"] > 0


def test_cli_gpus_argument_errors(capsys):
    assert main(["verify", "--kernel", "jacobi", "--variant", "threaded", "--gpus", "0"]) == 2


@pytest.mark.gpu
def test_fp64_probe_rate_is_plausible():
    """sb_fp64_probe: B200 FP64 is ~37 TFLOP/s counting an FMA as 2, i.e.
    ~18 T DP operations/s at boost clock; the probe must land near that."""
    from paper_1004_1741_b200.perf import fp64_peak

    ops = fp64_peak(iters=1 << 14)
    assert 8e12 < ops < 30e12, ops
