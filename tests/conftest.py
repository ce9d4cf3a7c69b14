import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer CPU test")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


# ---- full-size oracle results shared by the -m gpu parity tests (computed once per session)

@pytest.fixture(scope="session")
def c4_workload():
    import rpd_workloads as W
    return W.make_config("C4")


@pytest.fixture(scope="session")
def oracle_c4_chain(c4_workload):
    """The oracle's C3 full RPD and then its R11 partial update after each of the 10 C4
    batches: a list of (result, dirty tets) -- element 0 is the full RPD (dirty None)."""
    import numpy as np
    import oracle
    w = c4_workload
    prev = oracle.rpd_workload(w)
    chain = [(prev, None)]
    n_old = w.N
    for (sph, off, idx) in w.batches:
        prev, dirty = oracle.partial_update(prev, w.verts, w.tets, sph, off, idx, n_old)
        chain.append((prev, dirty))
        n_old = len(sph)
    return chain
