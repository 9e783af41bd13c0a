import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running oracle checks")
    config.addinivalue_line("markers", "sparse_path: run with the library's default Sinkhorn path "
                            "selection (small supports -> asot_sinkhorn_sparse.cu); other tests "
                            "pin the dense tensor-core / CUDA-core kernels with ASOT_SPARSE=0")


@pytest.fixture(autouse=True)
def _sinkhorn_path(request, monkeypatch):
    """The GPU tests written for the dense kernels keep exercising them (ASOT_SPARSE=0, read by
    the library on every call); tests marked sparse_path see the product's default selection."""
    if request.node.get_closest_marker("gpu") is None:
        pass   # CPU tests (and the bench.py subprocesses they start) see the environment as is
    elif request.node.get_closest_marker("sparse_path") is None:
        monkeypatch.setenv("ASOT_SPARSE", "0")
    else:
        monkeypatch.delenv("ASOT_SPARSE", raising=False)
    yield


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")) as f:
        return json.load(f)
