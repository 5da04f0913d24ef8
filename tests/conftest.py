import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    """Parse a golden text fixture into {section_name: ndarray}."""
    blocks, cur, rows = {}, None, []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line:
                continue
            if line.startswith("#"):
                tok = line[1:].strip()
                if tok and " " not in tok and ":" not in tok:
                    if cur is not None:
                        blocks[cur] = np.array(rows, dtype=np.float64)
                    cur, rows = tok, []
                continue
            rows.append([float(x) for x in line.split()])
    if cur is not None:
        blocks[cur] = np.array(rows, dtype=np.float64)
    elif rows:
        blocks["_"] = rows
    return blocks


@pytest.fixture
def golden():
    return load_golden
