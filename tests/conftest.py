import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
ASSETS = os.path.join(ROOT, "assets")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")


def _ensure_built():
    # The CPU oracle and the product library are built by __graft_entry__.build();
    # make is a no-op when they are current.
    if not os.path.exists(os.path.join(ROOT, "oracle", "liborc.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    if not os.path.exists(os.path.join(ROOT, "paper_2511_07418_b200", "libgraspgen_b200.so")):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_2511_07418_b200")],
                       check=True)


_ensure_built()


@pytest.fixture(scope="session")
def assets():
    return ASSETS


def asset(*parts):
    return os.path.join(ASSETS, *parts)


@pytest.fixture(scope="session")
def four_finger():
    import caller as lc
    import paper_2511_07418_b200 as lg
    return lc.load_hand(asset("hands", "four_finger.urdf"))


@pytest.fixture(scope="session")
def two_finger():
    import caller as lc
    import paper_2511_07418_b200 as lg
    return lc.load_hand(asset("hands", "two_finger.urdf"))


@pytest.fixture(scope="session")
def ctx():
    import caller as lc
    import paper_2511_07418_b200 as lg
    c = lg.Context(0)
    yield c
    c.close()


def cfg1(batch=64, passes=1, obj="sphere_r030.obj", hand="four_finger", **over):
    """Config 1: bundled hand + primitive object, reference cfg."""
    import caller as lc
    import paper_2511_07418_b200 as lg
    p = lc.parse_config(asset("configs", f"{hand}.cfg"), hand=asset("hands", f"{hand}.urdf"),
                        object=asset("objects", obj), batch=batch)
    p.passes = passes
    p.want_trace = 1
    for k, v in over.items():
        setattr(p, k, v)
    return p


def mismatched_fields(a, b, names=None):
    """Field-wise bitwise comparison of two structured arrays (padding bytes
    are not part of the record); returns {field: [row indices]}."""
    import numpy as np
    assert len(a) == len(b), (len(a), len(b))
    out = {}
    if len(a) == 0:
        return out
    for n in names or a.dtype.names:
        x = np.ascontiguousarray(a[n]).view(np.uint8).reshape(len(a), -1)
        y = np.ascontiguousarray(b[n]).view(np.uint8).reshape(len(b), -1)
        rows = np.nonzero((x != y).any(axis=1))[0]
        if len(rows):
            out[n] = rows.tolist()
    return out


def pytest_sessionfinish(session, exitstatus):
    """Under LG_CHECK_CANARY=1 every device buffer is guard-banded; fail the
    session when any kernel wrote past the end of one (test_canary.py)."""
    if os.environ.get("LG_CHECK_CANARY") != "1":
        return
    import paper_2511_07418_b200 as lg
    v = lg.lib().lg_debug_canary_violations()
    print(f"\ncanary_violations={v}")
    if v:
        session.exitstatus = 1
