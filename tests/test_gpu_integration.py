"""The B200 backend behind the REFERENCE's own C++ pipeline and plugin interfaces.

integration/_build/test_adapter links the reference's compiled sources (model_io, passes,
dfp::partition / lower_group / run_kernel, dnn::ProviderRegistry / candidates / heuristic_choice /
execute_choice, autodiff, run_reference) with integration/sol_b200_adapter.cpp: the reference
partitions and dispatches, the adapter's B200Backend (lower_group / interpret contract) runs every
fused unit and its B200Provider (dnn::KernelProvider) every heavy node on the GPU. Each unit is
checked against the reference's own implementation on the same inputs, and the outputs / gradients
against its f64 oracle (see integration/test_adapter.cpp for the bars)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_build", "test_adapter")


def _models():
    from paper_2003_10688_b200 import models
    return {
        "small_cnn": lambda: models.small_cnn(hw=32),
        "small_cnn_train": lambda: models.small_cnn(hw=16, train=True),
        "resnet18_tiny": lambda: models.resnet(18, hw=32, classes=10, width=8),
        "resnet18_tiny_train": lambda: models.resnet(18, hw=16, classes=10, width=8, train=True),
        "resnet50_tiny": lambda: models.resnet(50, hw=32, classes=10, width=8),
    }


CASES = [("small_cnn", 8, 0), ("small_cnn_train", 8, 1), ("resnet18_tiny", 4, 0), ("resnet18_tiny_train", 4, 1),
         ("resnet50_tiny", 2, 0)]


def test_adapter_binary_links_reference_and_backend():
    if not os.path.exists(BIN):
        pytest.skip("integration/_build/test_adapter not built (needs /root/reference at build time)")
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libsolb200.so" in out and "not found" not in out, out


@pytest.mark.gpu
@pytest.mark.parametrize("name,batch,train", CASES, ids=[c[0] for c in CASES])
def test_reference_pipeline_runs_on_b200(gpu, tmp_path, name, batch, train):
    from paper_2003_10688_b200 import graph
    if not os.path.exists(BIN):
        pytest.skip("integration/_build/test_adapter not built")
    g = _models()[name]()
    mj, wj = tmp_path / "model.json", tmp_path / "weights.solw"
    mj.write_text(graph.model_to_json(g))
    wj.write_bytes(graph.weights_to_bytes(g.params))
    r = subprocess.run([BIN, str(mj), str(wj), str(batch), str(train)], capture_output=True, text=True, timeout=300)
    line = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert line, (r.stdout, r.stderr)
    res = json.loads(line[-1])
    print(name, res)
    assert r.returncode == 0, res
    assert res["failures"] == 0 and res["dfp_units"] > 0 and res["heavy_units"] > 0
