import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def restatement():
    import oracle

    oracle.build(reference=False)
    return oracle.Restatement()


@pytest.fixture(scope="session")
def reference():
    import oracle

    if not os.path.exists(oracle.REF_SO):
        if os.path.isdir(oracle.REF_SRC):
            oracle.build(reference=True)
        else:
            pytest.skip("compiled reference (oracle/_ref) not available")
    return oracle.Reference()


@pytest.fixture(scope="session")
def plmss():
    import paper_2303_15491_b200 as P
    from paper_2303_15491_b200 import _build

    if not os.path.exists(_build.LIB):
        _build.build_cuda()
    return P


@pytest.fixture(scope="session")
def gpu(plmss):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return plmss.default_context(0)


def golden_cases():
    return sorted(f[5:-4] for f in os.listdir(GOLDEN) if f.startswith("case_") and f.endswith(".npz"))


def load_case(name):
    return dict(np.load(os.path.join(GOLDEN, f"case_{name}.npz")))
