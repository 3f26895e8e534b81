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
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture
def fe_opts():
    """Set libfeb200 implementation options (fe_set_option) for one test; restored after it.
    fe_opts(matrix_impl="dense", max_ctas=3) -- names / values as paper_2107_04121_b200.options."""
    import paper_2107_04121_b200 as fe
    saved = fe.get_options()

    def set_(**kw):
        fe.options(**kw).__enter__()

    yield set_
    for k, v in saved.items():
        fe.fe_set_option(fe._OPT_NAMES[k], v)
