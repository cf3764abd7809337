import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) GPU")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _have_gpu() -> bool:
    try:
        from paper_2512_00398_b200._native import device_count

        return device_count() > 0
    except Exception:
        return False


HAVE_GPU = _have_gpu()


def pytest_collection_modifyitems(config, items):
    if HAVE_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def ref():
    """The compiled reference library (oracle/_ref), if it was built."""
    from oracle import pyoracle

    if not pyoracle.REF_SO.exists():
        pytest.skip("reference library not built (oracle/_ref)")
    return pyoracle.Reference()


@pytest.fixture(scope="session")
def port():
    from oracle import pyoracle

    if not pyoracle.PORT_SO.exists():
        pyoracle.build()
    return pyoracle.Port()


@pytest.fixture(scope="session")
def engine():
    from paper_2512_00398_b200.engine import Engine

    eng = Engine(0)
    yield eng
    eng.close()


@pytest.fixture(scope="session")
def abl_engine():
    """A context of libpgb200_ablations.so: the PGB_* switchable alternatives (DESIGN.md
    section 10), compared against the product library's default path."""
    from paper_2512_00398_b200.engine import Engine

    eng = Engine(0, ablations=True)
    yield eng
    eng.close()
