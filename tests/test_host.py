"""Host-side logic of the drop-in (CPU only, no compute calls).

Validation semantics mirror the reference's TestValidation
(pkg/tests/test_engine.py:259-290); the value maps that carry reduced
precision and adaptive topologies are checked against the reference's own
outputs; the C-ABI library must load and export every symbol the header
declares.
"""

import re
from pathlib import Path

import numpy as np
import pytest

import paper_1105_3829_b200 as mtb
from oracle import oracle as O
from paper_1105_3829_b200 import _lib
from tests import golden_data as G

ROOT = Path(__file__).resolve().parents[1]


def random_image(rng, h, w, bit_depth=8):
    return mtb.GrayImage(
        rng.integers(0, 1 << bit_depth, size=(h, w)).astype(
            np.uint8 if bit_depth == 8 else np.uint16), bit_depth)


# ---------------------------------------------------------------- C ABI

def test_library_exports_every_header_symbol():
    header = (ROOT / "include" / "medtree_b200.h").read_text()
    declared = set(re.findall(r"\b(mtb_\w+)\s*\(", header))
    assert declared == set(_lib.EXPORTS)
    lib = _lib.load()
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.mtb_version() >= 1


def test_abi_rejects_invalid_arguments_without_device():
    lib = _lib.load()
    dummy = 1 << 20  # never dereferenced: validation precedes any CUDA call
    # window too large for a 4x4 image (validation.py:24-28)
    rc = lib.mtb_median_u8(dummy, 4, 0, 4, dummy, 4, 4, 4, 0, 4, 5, 61, None, 0, None)
    assert rc == _lib.MTB_E_INVAL
    assert b"too large" in lib.mtb_last_error()
    # rank outside [1, n^2] (validation.py:45-46)
    rc = lib.mtb_median_u8(dummy, 8, 0, 8, dummy, 8, 8, 8, 0, 8, 1, 10, None, 0, None)
    assert rc == _lib.MTB_E_INVAL and b"rank" in lib.mtb_last_error()
    # slab source rows do not cover the halo
    rc = lib.mtb_median_u16(dummy, 8, 2, 4, dummy, 8, 16, 8, 2, 6, 1, 5, None, 0, None)
    assert rc == _lib.MTB_E_INVAL and b"halo" in lib.mtb_last_error()
    rc = lib.mtb_median_u8(None, 8, 0, 8, dummy, 8, 8, 8, 0, 8, 1, 5, None, 0, None)
    assert rc == _lib.MTB_E_INVAL
    rc = lib.mtb_filter_host(dummy, dummy, 12, 8, 8, 1, 5, None, 0)
    assert rc == _lib.MTB_E_INVAL and b"bit_depth" in lib.mtb_last_error()
    rc = lib.mtb_filter_host_frames(dummy, dummy, dummy, None, 2, 12, 8, 8, None, 0)
    assert rc == _lib.MTB_E_INVAL and b"bit_depth" in lib.mtb_last_error()
    rc = lib.mtb_filter_host_frames(None, dummy, dummy, None, 2, 8, 8, 8, None, 0)
    assert rc == _lib.MTB_E_INVAL and b"null" in lib.mtb_last_error()
    assert lib.mtb_filter_host_frames(None, None, None, None, 0, 8, 8, 8, None, 0) == _lib.MTB_OK
    # host rows entry: its own checks run before any device call
    rc = lib.mtb_filter_host_rows(dummy, dummy, 12, 8, 8, 0, 8, 1, 5, None, 0, -1)
    assert rc == _lib.MTB_E_INVAL and b"bit_depth" in lib.mtb_last_error()
    rc = lib.mtb_filter_host_rows(dummy, dummy, 8, 8, 8, 3, 9, 1, 5, None, 0, -1)
    assert rc == _lib.MTB_E_INVAL and b"row range" in lib.mtb_last_error()
    rc = lib.mtb_filter_host_rows(None, dummy, 8, 8, 8, 0, 8, 1, 5, None, 0, -1)
    assert rc == _lib.MTB_E_INVAL and b"null" in lib.mtb_last_error()
    assert lib.mtb_filter_host_rows(dummy, dummy, 8, 8, 8, 4, 4, 1, 5, None, 0, -1) == _lib.MTB_OK


def test_host_entries_check_lut_length():
    """A value map must hold 2^bit_depth entries (the C host entries copy
    that many from the pointer): a short one is rejected in Python."""
    px16 = np.zeros((8, 8), np.uint16)
    with pytest.raises(ValueError, match="2\\^16"):
        mtb.filter_host_buffer(px16, 1, lut=np.arange(256, dtype=np.uint16))
    with pytest.raises(ValueError, match="2\\^8"):
        mtb.filter_host_frames([np.zeros((8, 8), np.uint8)], 1, lut=np.arange(16, dtype=np.uint8))


def test_host_frames_validates_before_any_device_call():
    px = np.zeros((8, 8), np.uint8)
    with pytest.raises(ValueError, match="shape and dtype"):
        mtb.filter_host_frames([px, np.zeros((8, 9), np.uint8)], 1)
    with pytest.raises(ValueError, match="one radius per frame"):
        mtb.filter_host_frames([px, px], [1, 2, 3])
    with pytest.raises(ValueError, match="odd integer"):
        mtb.filter_host_frames([px], 0)
    assert mtb.filter_host_frames([], 3) == []


# ----------------------------------------------------------- validation

class TestValidation:
    def test_even_window_rejected(self, rng):
        with pytest.raises(ValueError):
            mtb.filter_image(random_image(rng, 8, 8), 4)

    def test_window_one_rejected(self, rng):
        with pytest.raises(ValueError):
            mtb.filter_image(random_image(rng, 8, 8), 1)

    def test_window_too_large(self, rng):
        with pytest.raises(ValueError, match="too large"):
            mtb.filter_image(random_image(rng, 4, 4), 11)

    def test_bad_rank(self, rng):
        image = random_image(rng, 8, 8)
        for bad in (0, 10):
            with pytest.raises(ValueError):
                mtb.filter_image(image, 3, rank=bad)
        with pytest.raises(ValueError):
            mtb.filter_image(image, 3, rank=5, percentile=0.5)
        with pytest.raises(ValueError):
            mtb.filter_image(image, 3, percentile=0.0)

    def test_bad_max_error(self, rng):
        with pytest.raises(ValueError):
            mtb.filter_image(random_image(rng, 8, 8), 3, max_error=0)

    def test_bad_mode(self, rng):
        with pytest.raises(ValueError):
            mtb.filter_image(random_image(rng, 8, 8), 3, mode="bogus")

    def test_bad_bands(self, rng):
        with pytest.raises(ValueError):
            mtb.filter_image(random_image(rng, 8, 8), 3, bands=0)

    def test_topology_depth_mismatch(self, rng):
        with pytest.raises(ValueError):
            mtb.filter_image(random_image(rng, 8, 8, 16), 3, topology=mtb.uniform_topology(8))

    def test_profile_length_checked(self, rng):
        with pytest.raises(ValueError):
            mtb.filter_image(random_image(rng, 8, 8), 3, mode="adaptive",
                             profile=mtb.FrequencyProfile(np.ones(64)))

    def test_gray_image_rules(self):
        with pytest.raises(ValueError):
            mtb.GrayImage(np.zeros((0, 3), dtype=np.uint8))
        with pytest.raises(ValueError):
            mtb.GrayImage(np.zeros((3, 3), dtype=np.float32))
        with pytest.raises(ValueError):
            mtb.GrayImage(np.full((3, 3), 256, dtype=np.int64), 8)
        assert mtb.GrayImage(np.zeros((2, 2), dtype=np.int64)).bit_depth == 16
        assert mtb.GrayImage(np.zeros((2, 2), dtype=np.uint8)).bit_depth == 8

    def test_resolve_rank_matches_reference_rules(self):
        assert mtb.resolve_rank(3) == 5
        assert mtb.resolve_rank(11) == 61
        assert mtb.resolve_rank(3, percentile=1.0 / 9.0) == 1
        assert mtb.resolve_rank(5, percentile=0.5) == 13


# ------------------------------------------------------------ value maps

@pytest.mark.parametrize("d", [8, 16])
@pytest.mark.parametrize("max_error", [1, 2, 3, 16, 20, 1000, 1 << 17])
def test_uniform_value_map_is_reference_quantization(d, max_error):
    lut = mtb.value_map(mtb.uniform_topology(d), max_error)
    v = np.arange(1 << d, dtype=np.uint8 if d == 8 else np.uint16)
    expect = O.quantize_reference(v, d, max_error)
    got = v if lut is None else lut
    assert np.array_equal(got, expect)


@pytest.mark.parametrize("item", list(G.topologies()), ids=lambda t: t[0])
def test_product_topology_builder_matches_reference(item):
    name, arr = item
    img = mtb.GrayImage(arr["px"])
    topo = mtb.resolve_topology(img, int(arr["n"]), "adaptive")
    for key in ("up", "leaf", "span", "lo"):
        assert np.array_equal(getattr(topo, key), arr[key]), key


@pytest.mark.parametrize("case", [c for c in G.small_cases()
                                  if c[0]["mode"] == "adaptive" and c[0]["max_error"] > 1],
                         ids=lambda c: f"case{c[0]['idx']}")
def test_adaptive_value_map_reproduces_reference(case):
    meta, px, ref = case
    n = meta["n"]
    img = mtb.GrayImage(px, meta["bit_depth"])
    topo = mtb.resolve_topology(img, n, "adaptive")
    lut = mtb.value_map(topo, meta["max_error"])
    exact = O.sort_filter(px, n)
    got = exact if lut is None else lut[exact]
    assert np.array_equal(got, ref)


def test_no_cpu_fallback_without_device(rng):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        mtb.filter_image(random_image(rng, 8, 8), 3)
