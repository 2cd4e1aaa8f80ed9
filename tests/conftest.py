import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the CUDA extension")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(GOLDEN, "values.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def lm_pair():
    """The synthetic 4-gram LM (c3-c5) as a device handle, an oracle handle, and its path."""
    import oracle
    import paper_2508_07315_b200 as F
    import synth
    path = synth.arpa_file(V=1024)
    return F.LM(path, 1024, device=0), oracle.LM(path, 1024), path


@pytest.fixture(scope="session")
def bt_pair():
    """The 1000 synthetic phrases (c4, c5) as device and oracle boosting handles."""
    import oracle
    import paper_2508_07315_b200 as F
    import synth
    ph = synth.phrases(1024)
    return F.Boost(ph, 1.0, 1024, device=0), oracle.Boost(ph, 1.0, 1024), ph
