"""Every hub-walk schedule gives the oracle's passes bit for bit: cluster
pairs and quads, cooperative walks for all or only the big hubs, the
per-CTA phase for the rest, and the one-CTA-per-hub fallback (scan.cu
k_scan_hub / k_scan_spec<32, true, 4>)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))

MODES = [
    {},                                                     # defaults
    {"RNNDG_HUB": "0"},                                     # one CTA per hub
    {"RNNDG_HUB": "2", "RNNDG_COOP_ALL": "0"},              # big hubs coop, rest per CTA
    {"RNNDG_HUB": "4", "RNNDG_COOP_ALL": "0", "RNNDG_BIG_HUB": "256"},  # all hubs coop (quads)
    {"RNNDG_HUB": "4", "RNNDG_COOP_ALL": "0", "RNNDG_BIG_HUB": "0"},    # no cooperative walks
]


@pytest.mark.parametrize("env", MODES, ids=lambda e: ",".join(f"{k[6:]}={v}" for k, v in e.items()) or "default")
def test_hub_modes_match_oracle(env):
    full = dict(os.environ, **env)
    r = subprocess.run([sys.executable, os.path.join(HERE, "hub_case.py"), "400"], env=full,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
