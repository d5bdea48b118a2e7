import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a) and the built libepg.so")


def golden(name):
    with open(os.path.join(HERE, "golden", name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def mesh_c1():
    from synth import config_mesh
    return config_mesh("c1")


@pytest.fixture(scope="session")
def small_mesh():
    """A few thousand cells: several 256/1024-edge partitions plus a ragged tail."""
    from synth import kuhn_mesh
    return kuhn_mesh(nbox=9, n_keep=3_901)
