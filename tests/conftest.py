import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))

try:
    from hypothesis import settings

    settings.register_profile("ci", derandomize=True, deadline=None)
    settings.load_profile("ci")
except ImportError:  # pragma: no cover
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    # the C-ABI tests load libcrossover.so: build it (nvcc cross-compiles, no GPU needed) when a
    # fresh checkout has none or its sources changed -- the product itself never builds on import
    try:
        from paper_2103_07974_b200 import _build

        if _build.needs_rebuild():
            _build.build()
    except Exception as exc:  # noqa: BLE001 - no nvcc: the tests that need the library will say so
        print(f"conftest: libcrossover.so not built ({exc})", file=sys.stderr)


@pytest.fixture(scope="session")
def schedule_golden():
    return json.loads((GOLDEN / "schedule.json").read_text())["cases"]


@pytest.fixture(scope="session")
def equivalence_golden():
    meta = json.loads((GOLDEN / "equivalence_meta.json").read_text())
    arrays = dict(np.load(GOLDEN / "equivalence.npz"))
    return meta, arrays


@pytest.fixture(scope="session")
def fixtures_golden():
    return json.loads((GOLDEN / "fixtures.json").read_text())


@pytest.fixture(scope="session")
def cuda_device():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)
