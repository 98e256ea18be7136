"""Loader for the reference-generated fixtures in tests/golden/."""

import hashlib
import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def small_cases():
    with open(os.path.join(HERE, "small_cases.json")) as fh:
        meta = json.load(fh)
    data = np.load(os.path.join(HERE, "small_cases.npz"))
    for m in meta:
        i = m["idx"]
        yield m, data[f"in{i}"], data[f"out{i}"]


def digests():
    with open(os.path.join(HERE, "digests.json")) as fh:
        return json.load(fh)


_FULL = None


def fullsize_digests():
    """SHA-256 of the reference's outputs at the BASELINE sizes
    (make_fullsize_digests.py)."""
    global _FULL
    if _FULL is None:
        with open(os.path.join(HERE, "fullsize_digests.json")) as fh:
            _FULL = json.load(fh)
    return _FULL


def topologies():
    data = np.load(os.path.join(HERE, "topologies.npz"))
    names = sorted({k.rsplit("_", 1)[0] for k in data.files})
    for name in names:
        yield name, {k.rsplit("_", 1)[1]: data[k] for k in data.files if k.rsplit("_", 1)[0] == name}


# BASELINE.md "Golden vector (config 1)"
CFG1_INPUT_SHA = "d022786ba1ea558754e863dc43f95a8a909104fa3e5d4379853b7f4e2a26f5e2"
CFG1_OUTPUT_SHA = "21beb9a65da6cf0928c6271b3b7f2e62d8f55c3c82fe72962735daa3f7b910ba"
CFG1_FIRST8 = [121, 123, 130, 130, 144, 163, 163, 184]
