import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); parity of the CUDA path vs the oracle")
    config.addinivalue_line("markers", "slow: large inputs (seconds)")


@pytest.fixture(scope="session")
def engine():
    from paper_1710_06189_b200 import texforge as tf
    return tf.default_engine()


@pytest.fixture(scope="session")
def small_cases():
    import numpy as np
    z = np.load(os.path.join(GOLDEN, "small_cases.npz"))
    meta, pix, po, cnt, co = z["meta"], z["pixels"], z["pix_off"], z["counts"], z["cnt_off"]
    cases = []
    for i, m in enumerate(meta):
        w, h, L, d, th, pl = (int(x) for x in m)
        cases.append(dict(w=w, h=h, L=L, d=d, theta=th, pixel_levels=pl, pixels=pix[po[i]:po[i + 1]],
                          counts=cnt[co[i]:co[i + 1]], probs=z["probs"][co[i]:co[i + 1]], feats=z["feats"][i]))
    return cases


@pytest.fixture(scope="session")
def golden_hashes():
    import json
    with open(os.path.join(GOLDEN, "golden_hashes.json")) as f:
        return json.load(f)
