import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def facts():
    return load_golden("paper_facts.json")


@pytest.fixture(scope="session")
def spec():
    return load_golden("spec_examples.json")


@pytest.fixture
def knobs():
    """knobs(cta_group=1, mod_split=0, ...) sets the library's tuning knobs for the calling
    thread (OZ2_TUNE_*, schedule only); each knob gets its previous value back after the
    test."""
    import paper_2603_10634_b200 as P
    prev = {}

    def set_(**kw):
        for k, v in kw.items():
            prev.setdefault(k, P.oz2_get_tuning(k))
            assert P.oz2_set_tuning(k, int(v)) == 0, (k, v)
    yield set_
    for k, v in prev.items():
        P.oz2_set_tuning(k, v)
