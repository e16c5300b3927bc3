import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


RANDOM_CASES = [
    "smoke_f64", "smoke_f32", "t1_w1_f32", "t2_w3_f32", "t257_b2_n4_f32",
    "t1000_b3_n7_f32", "t300_b1_n130_f32", "t513_b2_n64_f32",
    "t2000_b1_n8_near1_f32", "t4096_b1_n16_f32", "t700_b1_n9_f64",
    "t129_b2_n66_f64",
]


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()
