"""bench_cli host operations (SPEC.md bench_cli: efficiency, scaling_report,
RunConfig / MetricsRecord CSV) and a GPU run_benchmark / verify check."""
import csv
import io

import pytest

from paper_2312_13094_b200 import bench_cli as BC
from paper_2312_13094_b200 import distfield as DF
from paper_2312_13094_b200 import decomposition as DC


def test_efficiency_examples():
    assert BC.efficiency([1.0, 2.0, 4.0]) == [100.0, 100.0, 100.0]
    assert BC.efficiency([1.0, 1.0]) == [100.0, 50.0]


def test_scaling_report_weak_and_strong():
    rows = BC.scaling_report("weak", (32, 32, 32), [1, 2, 4])
    assert [r["shape"] for r in rows] == [(32, 32, 32), (64, 32, 32), (64, 64, 32)]
    rows = BC.scaling_report("strong", (64, 64, 64), [1, 2, 4, 8])
    assert {r["shape"] for r in rows} == {(64, 64, 64)}
    with pytest.raises(ValueError):
        BC.scaling_report("sideways", (8, 8), [1])


def test_weak_series_interior_bytes_constant():
    """Interior-rank exchange volume per step is constant across the weak series."""
    vols = []
    for r, topo in ((64, (4, 4, 4)), (128, (8, 4, 4)), (256, (8, 8, 4))):
        shape = BC.scaling_report("weak", (32, 32, 32), [r])[0]["shape"]
        d = DC.Decomposition.create(shape, r, topo)
        interior = [k for k in range(r) if len(DF.diagonal_messages(d, k, (4, 4, 4))) == 26]
        vols.append({sum(m.volume for m in DF.diagonal_messages(d, k, (4, 4, 4)))
                     for k in interior})
    assert all(v == vols[0] and len(v) == 1 for v in vols), vols


def test_metrics_csv_round_trip():
    cfg = BC.RunConfig(kernel="diffusion", shape=(64, 64), sdo=2, steps=10)
    from dataclasses import asdict
    conf = asdict(cfg)
    conf.update(ranks=1, topology=(1, 1))
    rec = BC.MetricsRecord(conf, 0.5, 64 * 64 * 10 / 0.5 / 1e9, 0, 0, 12.5, 0.0)
    text = BC.to_csv([rec])
    rows = list(csv.DictReader(io.StringIO(text)))
    assert tuple(rows[0].keys()) == BC.CSV_COLUMNS
    assert rows[0]["shape"] == "64x64" and float(rows[0]["checksum"]) == 12.5
    assert float(rows[0]["gpts_per_s"]) == pytest.approx(64 * 64 * 10 / 0.5 / 1e9)


@pytest.mark.gpu
@pytest.mark.parametrize("kernel,shape,so", [("diffusion", (64, 64), 2),
                                             ("acoustic", (48, 40, 44), 8)])
def test_run_benchmark_deterministic_and_verified(kernel, shape, so):
    cfg = BC.RunConfig(kernel=kernel, shape=shape, sdo=so, steps=10, mode="full", check=True)
    a = BC.run_benchmark(cfg)
    b = BC.run_benchmark(cfg)
    assert a.checksum == b.checksum and a.checksum > 0
    assert a.max_diff == 0.0
    assert a.gpts_per_s == pytest.approx(
        (shape[0] * shape[1] * (shape[2] if len(shape) > 2 else 1)) * 9 / a.walltime_s / 1e9)


def test_cli_dump_plan(capsys):
    """`--dump-plan` prints the Listing-6/7-style tree (host only, no GPU)."""
    rc = BC.main(["--kernel", "acoustic", "--shape", "24,20,16", "--so", "4", "--mode", "full",
                  "--dump-plan"])
    out = capsys.readouterr().out
    assert rc == 0 and "<Callable Kernel>" in out and "Iteration time" in out


def test_cli_rejects_cpu_transports_and_rank_mismatch():
    with pytest.raises(SystemExit):
        BC.main(["--transport", "socket", "--dump-plan"])
    with pytest.raises(SystemExit):
        BC.main(["--ranks", "4", "--dump-plan", "--shape", "16,16,16", "--so", "4"])
