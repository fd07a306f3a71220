import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) CUDA device")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def codec_golden():
    return np.load(os.path.join(GOLDEN, "codec_layout.npz"))


@pytest.fixture(scope="session")
def attn_golden():
    return np.load(os.path.join(GOLDEN, "attention_cases.npz"))


def golden_cases(attn):
    """Decoded meta of every attention golden case."""
    out = {}
    for name in sorted({k.split("__")[0] for k in attn.files}):
        m = attn[name + "__meta"]
        out[name] = dict(
            grid=tuple(int(x) for x in m[0:3]), d=int(m[3]), tile=tuple(int(x) for x in m[4:7]),
            window=tuple(int(x) for x in m[7:10]), fmt=["e4m3", "e5m2"][int(m[10])], seed=int(m[11]),
            dist=["gaussian", "uniform", "heavy"][int(m[12])])
    return out


CASE_NAMES = ["c0_toy", "c0_toy_full", "small_d128", "tv120_d128", "tv240_d128", "tv240_heavy", "tv240_e5m2",
              "tv504_d128", "tv256_d64"]
