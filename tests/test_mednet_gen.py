"""The generated merge/select networks of k_mednet (tools/gen_mednet.py):
the committed header is the generator's output, and the networks select
the median of every window on random and tie-heavy inputs (CPU)."""

import pathlib
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))

import gen_mednet as G  # noqa: E402


def test_header_is_generator_output():
    out = subprocess.run([sys.executable, str(ROOT / "tools" / "gen_mednet.py")], capture_output=True,
                         text=True, check=True).stdout
    assert (ROOT / "paper_1105_3829_b200" / "csrc" / "mednet_gen.cuh").read_text() == out


def test_networks_select_the_median():
    # G.check raises on the first window whose network output is not the
    # median of its n*n values (value ranges 2, 3, 5 and 256)
    assert G.check(5, trials=1500) == 162
    assert G.check(7, trials=1500) == 400
