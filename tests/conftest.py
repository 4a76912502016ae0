import gzip
import json
import pathlib
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = pathlib.Path(__file__).parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA extension")


@pytest.fixture(scope="session")
def planner_golden():
    return json.loads(gzip.decompress((GOLDEN / "planner_golden.json.gz").read_bytes()))


@pytest.fixture(scope="session")
def uni8(planner_golden):
    from paper_2505_05856_b200.planner import graph_from_doc
    return graph_from_doc(planner_golden["cases"][0]["profile"])


@pytest.fixture(scope="session")
def tri4(planner_golden):
    from paper_2505_05856_b200.planner import graph_from_doc
    return graph_from_doc(planner_golden["cases"][1]["profile"])
