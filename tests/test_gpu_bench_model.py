"""The reference's bench_model (bench.hpp:246-414, paper Table 2 regime) on the
GPU at a reduced preset: every architecture's two-layer train step runs with
serial and parallel recurrences, the reference's 2e-4 serial/parallel guard
holds (the script exits otherwise), and the records carry the reference's
fields (events/s per mode, speedup)."""
import json
import os
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "scripts"))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def test_bench_model_reduced_preset(tmp_path):
    import bench_model
    out = tmp_path / "bm.json"
    recs = bench_model.main(["--bt", "4096", "--seq-lens", "16", "256", "4096", "--hidden", "64", "--reps", "2",
                             "--warmup", "1", "--out", str(out)])
    done = [r for r in recs if not r.get("skipped")]
    assert {r["arch"] for r in done} == {"gilr", "gilr-lstm", "qrnn-k2", "qrnn-k10"}
    for r in done:
        assert r["b"] * r["T"] == 4096
        assert r["serial"]["events_per_sec"] > 0 and r["parallel"]["events_per_sec"] > 0
        assert r["speedup"] == pytest.approx(r["serial"]["seconds"] / r["parallel"]["seconds"])
    # qrnn-k10 at T = 16 is computed; the reference skips only k > T
    assert any(r.get("skipped") for r in recs) is False
    saved = json.loads(out.read_text())
    assert len(saved["records"]) == len(recs)
    assert (tmp_path / "bm.md").exists()
