import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")
    config.addinivalue_line("markers", "slow: large-size parity (seconds to minutes)")


@pytest.fixture(scope="session")
def oracle():
    from oracle_bindings import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle_bindings import REF_SO, Ref
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return Ref()


def pytest_runtest_teardown(item, nextitem):
    # developer aid: DMTK_TEST_MEMLOG=<file> appends the device's free memory after every test
    path = os.environ.get("DMTK_TEST_MEMLOG")
    if not path:
        return
    try:
        import torch
        if not torch.cuda.is_available():
            return
        free, total = torch.cuda.mem_get_info()
        with open(path, "a") as f:
            f.write(f"{free / 2**30:8.2f} GiB free  torch_reserved {torch.cuda.memory_reserved() / 2**30:7.2f}  {item.nodeid}\n")
    except Exception:  # never fail a test over the log
        pass
