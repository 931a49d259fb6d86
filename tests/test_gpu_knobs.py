"""Every schedule knob that is kept gives the oracle's graph
and counters bit for bit: the Gram-filtered walk on / off / capped, the
short-list kernel's provisional depth, old-run rounds, list orders, the CUB
sort, the one-CTA-per-hub widths, the round-synchronous walk (bsp.cu), and --
on short rows -- the shared-memory walk (rowwalk.cu) on / capped / off, with
helper warps, other size classes and depths.  Each setting runs
tests/knob_case.py in its own process (the knobs are read once per process)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))

KNOBS = [
    {},
    {"RNNDG_GRAM": "128"},
    {"RNNDG_GRAM": "32"},
    {"RNNDG_GRAM": "64"},
    {"RNNDG_SPEC": "2"},
    {"RNNDG_SPEC": "4"},
    {"RNNDG_RUN": "0"},
    {"RNNDG_ORDER": "1"},
    {"RNNDG_ORDER": "2"},
    {"RNNDG_CUBSORT": "1"},
    {"RNNDG_HUB": "0", "RNNDG_LONG_W": "8"},
    {"RNNDG_HUB": "0", "RNNDG_LONG_W": "16"},
    {"RNNDG_UCAP": "128", "RNNDG_LS": "0"},
    # round-synchronous walk (bsp.cu): all lists finished inside their warps,
    # two / many rounds, a shorter cut-off, with deeper / shallower speculation,
    # without the side stream
    {"RNNDG_BSP": "1"},
    {"RNNDG_BSP": "2"},
    {"RNNDG_BSP": "8"},
    {"RNNDG_BSP": "64", "RNNDG_BSP_LEN": "40"},
    {"RNNDG_BSP": "6", "RNNDG_SPEC": "4"},
    {"RNNDG_BSP": "6", "RNNDG_SPEC": "2", "RNNDG_BSP_STREAM": "0"},
    {"RNNDG_BSP": "12", "RNNDG_BSP_STREAM": "2"},
    # short rows (RNNDG_CASE_D sets the dimension of the `passes` case): the
    # shared-memory walk (rowwalk.cu) on, capped, off, with other depths
    {"RNNDG_CASE_D": "96"},
    {"RNNDG_CASE_D": "128"},
    {"RNNDG_CASE_D": "96", "RNNDG_ROWWALK": "32"},
    {"RNNDG_CASE_D": "128", "RNNDG_ROWWALK": "0"},
    {"RNNDG_CASE_D": "96", "RNNDG_SPEC": "4"},
    {"RNNDG_CASE_D": "96", "RNNDG_SPEC": "2", "RNNDG_ROWWALK": "64"},
    {"RNNDG_CASE_D": "144"},
    # ... with helper warps per list, other size classes (up to 128 entries:
    # the 4-word masks), a small shared-memory budget
    {"RNNDG_CASE_D": "96", "RNNDG_ROWWALK_NW": "2"},
    {"RNNDG_CASE_D": "128", "RNNDG_ROWWALK_NW": "4", "RNNDG_ROWWALK": "128"},
    {"RNNDG_CASE_D": "96", "RNNDG_ROWWALK_CLS": "8,16,24,40", "RNNDG_ROWWALK_SMEM": "64"},
    {"RNNDG_CASE_D": "32", "RNNDG_ROWWALK": "128", "RNNDG_ROWWALK_D": "4"},
]


def _id(env):
    return ",".join(f"{k[6:]}={v}" for k, v in env.items()) or "default"


@pytest.mark.parametrize("case", ["passes", "build"])
@pytest.mark.parametrize("env", KNOBS, ids=_id)
def test_knob_matches_oracle(env, case):
    full = dict(os.environ, **env)
    r = subprocess.run([sys.executable, os.path.join(HERE, "knob_case.py"), case], env=full,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("tab", ["4", "6"])
def test_search_bitmap_rerun_matches(tab):
    """A seen-set table too small for the queries (RNNDG_SEARCH_TAB forces
    2^4 / 2^6 ids): every query overflows it and is re-run with the n-bit
    map (eval.cu k_search), so the search parity cases must still pass."""
    full = dict(os.environ, RNNDG_SEARCH_TAB=tab)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(HERE, "test_gpu_parity.py"), "-k", "search"],
                       env=full, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.slow
def test_gram_walk_fullsize_equals_reference():
    """The tensor-core Gram walk (RNNDG_GRAM=128) at the BASELINE sizes:
    the C3 1M x 960 and C4 1M x 96 builds byte-identical to the reference's
    (tests/test_gpu_fullsize.py in a process with the walk on)."""
    full = dict(os.environ, RNNDG_GRAM="128")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(HERE, "test_gpu_fullsize.py"), "-k", "C3 or C4"],
                       env=full, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
