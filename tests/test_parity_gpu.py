"""GPU parity: the CUDA path against the reference (golden fixtures) and
the CPU oracle.  Bit-exact everywhere (integer work, no tolerance).

Mirrors the reference's exactness matrix (pkg/tests/test_engine.py:25-99,
:243-256; pkg/tests/test_acceptance.py:46-93, :186-233) and adds the five
BASELINE configs: reduced-size digests and FULL-SIZE digests (every config
at the size BASELINE.json names, every radius of its sweep, config 5 as
the 64-image batch) recorded from the reference's own filter_image by
tests/golden/make_golden.py and make_fullsize_digests.py.
"""

import numpy as np
import pytest

import paper_1105_3829_b200 as mtb
import workloads
from oracle import oracle as O
from tests import golden_data as G

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _device():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _ref_args(meta):
    return dict(rank=meta["rank"], percentile=meta["percentile"],
                max_error=meta["max_error"], mode=meta["mode"])


@pytest.mark.parametrize("case", list(G.small_cases()), ids=lambda c: f"case{c[0]['idx']}")
def test_golden_small_cases(case):
    meta, px, ref = case
    out, ops = mtb.filter_image(mtb.GrayImage(px, meta["bit_depth"]), meta["n"],
                                **_ref_args(meta))
    assert out.pixels.dtype == ref.dtype
    assert np.array_equal(out.pixels, ref)
    assert ops.pixels == px.size


def test_cfg1_golden_digest():
    px = workloads.cfg1_uniform_u8()
    out, _ = mtb.filter_image(px, 11)
    assert G.sha(out.pixels) == G.CFG1_OUTPUT_SHA
    assert out.pixels[0, :8].tolist() == G.CFG1_FIRST8


def _digest_inputs():
    px2 = workloads.cfg2_blur_sp_u8(512, 512)
    px3 = workloads.cfg3_uniform_u16(192, 160)
    px4 = workloads.cfg4_three_gauss_u16(160, 192)
    b5 = workloads.cfg5_batch_u8(4, 256, 256)
    items = []
    for name, rec in sorted(G.digests().items()):
        if name.startswith("cfg2"):
            items.append((name, px2, rec))
        elif name.startswith("cfg3"):
            items.append((name, px3, rec))
        elif name.startswith("cfg4"):
            items.append((name, px4, rec))
        elif name.startswith("cfg5"):
            items.append((name, b5[int(name.split("img")[1].split("_")[0])], rec))
    return items


@pytest.mark.parametrize("item", _digest_inputs(), ids=lambda t: t[0])
def test_config_shaped_digests(item):
    name, px, rec = item
    out, _ = mtb.filter_image(px, rec["n"], mode=rec["mode"])
    assert G.sha(out.pixels) == rec["output"]


# ----------------------------------------------------- edge cases (test_engine.py)

@pytest.mark.parametrize("rank", [1, 5, 9])
def test_arbitrary_ranks(rng, rank):
    px = rng.integers(0, 256, (16, 14), dtype=np.uint8)
    out, _ = mtb.filter_image(px, 3, rank=rank)
    assert np.array_equal(out.pixels, O.sort_filter(px, 3, rank))


def test_min_max_percentiles(rng):
    from numpy.lib.stride_tricks import sliding_window_view

    px = rng.integers(0, 256, (12, 15), dtype=np.uint8)
    lo, _ = mtb.filter_image(px, 3, percentile=1.0 / 9.0)
    hi, _ = mtb.filter_image(px, 3, percentile=1.0)
    wins = sliding_window_view(np.pad(px, 1, mode="edge"), (3, 3)).reshape(12, 15, 9)
    assert np.array_equal(lo.pixels, wins.min(axis=2))
    assert np.array_equal(hi.pixels, wins.max(axis=2))


def test_constant_and_outlier():
    out, _ = mtb.filter_image(np.full((10, 10), 99, dtype=np.uint8), 5)
    assert (out.pixels == 99).all()
    px = np.full((3, 3), 10, dtype=np.uint8)
    px[1, 1] = 250
    assert mtb.filter_image(px, 3)[0].pixels[1, 1] == 10
    assert mtb.filter_image(np.array([[123]], dtype=np.uint8), 3)[0].pixels[0, 0] == 123


def test_checkerboard_majority():
    px = (np.indices((12, 12)).sum(axis=0) % 2 * 200).astype(np.uint8)
    out, _ = mtb.filter_image(px, 3, rank=5)
    assert np.array_equal(out.pixels[1:-1, 1:-1], px[1:-1, 1:-1])
    assert np.array_equal(out.pixels, O.sort_filter(px, 3, 5))


@pytest.mark.parametrize("shape", [(1, 40), (40, 1), (2, 19), (19, 2), (1, 1), (1, 300), (300, 1)])
@pytest.mark.parametrize("d", [8, 16])
def test_degenerate_geometries(rng, shape, d):
    px = rng.integers(0, 1 << d, size=shape).astype(np.uint8 if d == 8 else np.uint16)
    for n in (3, 2 * min(shape) + 1):
        if n < 3:
            continue
        out, _ = mtb.filter_image(px, n)
        assert np.array_equal(out.pixels, O.sort_filter(px, n)), n


@pytest.mark.parametrize("d", [8, 16])
def test_window_larger_than_image(rng, d):
    px = rng.integers(0, 1 << d, size=(7, 12)).astype(np.uint8 if d == 8 else np.uint16)
    for n in (9, 13, 15):
        out, _ = mtb.filter_image(px, n)
        assert np.array_equal(out.pixels, O.sort_filter(px, n)), n


def test_wide_counters_huge_window(rng):
    # n^2 > 65535 selects 32-bit window counters
    px = rng.integers(0, 256, (140, 300), dtype=np.uint8)
    n = 259
    out, _ = mtb.filter_image(px, n)
    assert np.array_equal(out.pixels, O.iot_filter(px, n))
    px16 = rng.integers(0, 65536, (130, 140)).astype(np.uint16)
    out16, _ = mtb.filter_image(px16, 257, rank=3)
    assert np.array_equal(out16.pixels, O.iot_filter(px16, 257, 3))


@pytest.mark.parametrize("max_error", [2, 16, 64, 1000])
def test_reduced_precision_uniform_16bit(rng, max_error):
    px = rng.integers(0, 65536, (24, 24)).astype(np.uint16)
    out, _ = mtb.filter_image(px, 5, max_error=max_error)
    assert np.array_equal(out.pixels, O.iot_filter(px, 5, max_error=max_error))
    exact = O.sort_filter(px, 5)
    diff = exact.astype(np.int64) - out.pixels.astype(np.int64)
    assert (diff >= 0).all() and diff.max() < max_error


@pytest.mark.parametrize("max_error", [4, 16])
def test_reduced_precision_adaptive_8bit(max_error):
    px = workloads.cfg4_three_gauss_u16(40, 36) >> 4
    px = px.astype(np.uint8)
    out, _ = mtb.filter_image(px, 7, mode="adaptive", max_error=max_error)
    ref = O.iot_filter(px, 7, mode="adaptive", max_error=max_error)
    assert np.array_equal(out.pixels, ref)


@pytest.mark.parametrize("bands", [2, 3, 7, 64])
def test_bands_identical(rng, bands):
    px = rng.integers(0, 256, (33, 21), dtype=np.uint8)
    single, _ = mtb.filter_image(px, 5)
    banded, _ = mtb.filter_image(px, 5, bands=bands)
    assert np.array_equal(single.pixels, banded.pixels)


def test_slab_calls_reassemble_the_frame(rng):
    """Row slabs with halos from the host copy == one full-frame call
    (the multi-GPU decomposition, exercised on one device)."""
    px = rng.integers(0, 65536, (97, 75)).astype(np.uint16)
    r = 6
    full = mtb.rank_filter(torch.from_numpy(px).cuda(), r).cpu().numpy()
    H = px.shape[0]
    edges = [0, 13, 40, 41, 80, 97]
    got = np.empty_like(px)
    for a, b in zip(edges[:-1], edges[1:]):
        top, bot = max(0, a - r), min(H, b + r)
        src = torch.from_numpy(np.ascontiguousarray(px[top:bot])).cuda()
        got[a:b] = mtb.rank_filter(src, r, rows=(a, b), src_row0=top, height=H).cpu().numpy()
    assert np.array_equal(got, full)
    assert np.array_equal(full, O.iot_filter(px, 2 * r + 1))


def test_batch_matches_single_images():
    b5 = workloads.cfg5_batch_u8(4, 192, 160)
    t = torch.from_numpy(b5).cuda()
    for r in (7, 25):
        out = mtb.rank_filter(t, r).cpu().numpy()
        for i in range(b5.shape[0]):
            assert np.array_equal(out[i], O.iot_filter(b5[i], 2 * r + 1)), (r, i)


def test_host_buffer_entry_point(rng):
    px = rng.integers(0, 256, (50, 61), dtype=np.uint8)
    assert np.array_equal(mtb.filter_host_buffer(px, 4), O.iot_filter(px, 9))
    px16 = rng.integers(0, 65536, (40, 33)).astype(np.uint16)
    lut = mtb.value_map(mtb.uniform_topology(16), 16)
    assert np.array_equal(mtb.filter_host_buffer(px16, 3, lut=lut),
                          O.iot_filter(px16, 7, max_error=16))


@pytest.mark.parametrize("stream", ["1", "0", "2", "3", "4"])
def test_host_frames_sequence(rng, stream, monkeypatch):
    """mtb_filter_host_frames: a sequence longer than the buffer ring (3),
    mixed radii and ranks, 8- and 16-bit, pinned and pageable frames, a value
    map -- every frame equal to its own oracle result."""
    monkeypatch.setenv("MTB_FRAMES_STREAM", stream)
    frames = [workloads.cfg2_blur_sp_u8(300, 150) for i in range(7)]
    frames = [np.ascontiguousarray(np.roll(f, 5 * i, axis=1)) for i, f in enumerate(frames)]
    radii = [1, 3, 7, 2, 15, 31, 5]
    pinned = [torch.from_numpy(f).pin_memory().numpy() for f in frames]
    outs = mtb.filter_host_frames(pinned, radii)
    for f, r, o in zip(frames, radii, outs):
        assert np.array_equal(o, O.iot_filter(f, 2 * r + 1)), r
    ranks = [1, 49, 10, 25, 100, 1000, 121]
    outs = mtb.filter_host_frames(frames, radii, ranks=ranks)
    for f, r, k, o in zip(frames, radii, ranks, outs):
        assert np.array_equal(o, O.iot_filter(f, 2 * r + 1, k)), (r, k)
    f16 = [rng.integers(0, 65536, (260, 52)).astype(np.uint16) for _ in range(4)]
    lut = mtb.value_map(mtb.uniform_topology(16), 16)
    outs = mtb.filter_host_frames(f16, 3, lut=lut)
    for f, o in zip(f16, outs):
        assert np.array_equal(o, O.iot_filter(f, 7, max_error=16))


@pytest.mark.parametrize("perm", ["6,0,5,1,4,2,3", "0,1,2,3,4,5,6", "0,0,1,2,3,4,5", "junk"])
def test_host_frames_explicit_order(perm, monkeypatch):
    """MTB_FRAMES_PERM reorders the processing (invalid lists are ignored):
    every result still lands in its own output."""
    monkeypatch.setenv("MTB_FRAMES_PERM", perm)
    frames = [np.ascontiguousarray(np.roll(workloads.cfg2_blur_sp_u8(300, 150), 7 * i, axis=1)) for i in range(7)]
    radii = [3, 1, 15, 7, 2, 31, 5]
    outs = mtb.filter_host_frames(frames, radii)
    for f, r, o in zip(frames, radii, outs):
        assert np.array_equal(o, O.iot_filter(f, 2 * r + 1)), (perm, r)


@pytest.mark.parametrize("bits,r,bands,stream", [(8, 2, None, None), (8, 9, "3", None), (8, 40, None, None),
                                                 (16, 5, None, None), (16, 20, "5", None), (8, 3, "16", None),
                                                 (8, 2, None, "1"), (8, 40, None, "0"), (8, 70, None, "1"),
                                                 (16, 3, None, "1"), (16, 6, None, "1"), (8, 1, None, "1"),
                                                 (8, 1, "3", "0")])
def test_host_pipeline_bands(bits, r, bands, stream, monkeypatch):
    """mtb_filter_host overlaps copies with filtering -- row bands, or one
    streaming launch whose CTAs wait for their rows (stream memory ops);
    results must not depend on the mode or the band count (pinned and
    pageable buffers, caller-provided out)."""
    if bands:
        monkeypatch.setenv("MTB_HOST_BANDS", bands)
    if stream:
        monkeypatch.setenv("MTB_HOST_STREAM", stream)
    rng = np.random.default_rng(bits * 100 + r)
    # r = 1: W % 16 == 0 takes the TMA-staged 3x3 kernel (streaming case),
    # W = 333 the register one (banded case)
    H, W = 1300, (336 if (r == 1 and bands is None) else 333)
    if bits == 8:
        px = workloads.cfg2_blur_sp_u8(H, W, seed=r)
    else:
        px = (25000 + rng.normal(0, 500, (H, W))).clip(0, 65535).astype(np.uint16)
    tdt = torch.uint8 if bits == 8 else torch.uint16
    pin_src = torch.empty((H, W), dtype=tdt).pin_memory().numpy()
    pin_src[...] = px
    pin_out = torch.empty((H, W), dtype=tdt).pin_memory().numpy()
    got = mtb.filter_host_buffer(pin_src, r, out=pin_out)
    assert got is pin_out
    ref = O.iot_filter(px, 2 * r + 1)
    assert np.array_equal(pin_out, ref)
    assert np.array_equal(mtb.filter_host_buffer(px, r), ref)
    with pytest.raises(ValueError):
        mtb.filter_host_buffer(px, r, out=np.empty((H, W + 1), px.dtype))


# ------------------------------------------------ full-size BASELINE configs
# Every output byte of every config at its BASELINE size, hashed against the
# reference's own output (tests/golden/fullsize_digests.json).

_cache = {}


def _frame(key):
    if key not in _cache:
        _cache.clear()  # one large frame at a time
        gen = {"cfg2": workloads.cfg2_blur_sp_u8, "cfg3": workloads.cfg3_uniform_u16,
               "cfg4": workloads.cfg4_three_gauss_u16, "cfg5": workloads.cfg5_batch_u8}[key]
        _cache[key] = gen()
    return _cache[key]


def _full(name):
    rec = G.fullsize_digests()[name]
    return rec


@pytest.mark.parametrize("r", workloads.CONFIG_RADII[2])
def test_cfg2_full_size_digest(r):
    """Config 2 (4096^2 u8): the drop-in filter_image (pageable frame), the
    streaming host entry on a page-locked frame, and the device-resident
    entry -- all equal to the reference's full frame."""
    px = _frame("cfg2")
    rec = _full(f"cfg2_4096_r{r}")
    assert G.sha(px) == rec["input"]
    out, _ = mtb.filter_image(px, 2 * r + 1)
    assert G.sha(out.pixels) == rec["output"]
    pin = torch.from_numpy(px).pin_memory().numpy()
    pout = torch.empty(px.shape, dtype=torch.uint8).pin_memory().numpy()
    assert G.sha(mtb.filter_host_buffer(pin, r, out=pout)) == rec["output"]
    dev = mtb.rank_filter(torch.from_numpy(px).cuda(), r).cpu().numpy()
    assert G.sha(dev) == rec["output"]


@pytest.mark.parametrize("r", [80, 127])
def test_cfg2_full_size_digest_large_radii(r):
    """The config-2 frame beyond BASELINE's sweep, where the tcgen05 kernel
    (k_bandtc_u8) takes over: device-resident and streaming host entries
    against the reference's own full frame."""
    from paper_1105_3829_b200 import _lib

    px = _frame("cfg2")
    rec = _full(f"cfg2_4096_r{r}")
    assert G.sha(px) == rec["input"]
    dev = mtb.rank_filter(torch.from_numpy(px).cuda(), r).cpu().numpy()
    assert _lib.last_kernel().startswith("k_bandtc_u8"), _lib.last_kernel()
    assert G.sha(dev) == rec["output"]
    pin = torch.from_numpy(px).pin_memory().numpy()
    assert G.sha(mtb.filter_host_buffer(pin, r)) == rec["output"]


@pytest.mark.parametrize("r", workloads.CONFIG_RADII[3])
def test_cfg3_full_size_digest(r):
    """Config 3 (4096^2 u16 uniform): host entry and device-resident entry
    (whose 16-bit kernel choice is sampled on the device)."""
    px = _frame("cfg3")
    rec = _full(f"cfg3_4096_r{r}")
    assert G.sha(px) == rec["input"]
    out, _ = mtb.filter_image(px, 2 * r + 1)
    assert G.sha(out.pixels) == rec["output"]
    dev = mtb.rank_filter(torch.from_numpy(px).cuda(), r).cpu().numpy()
    assert G.sha(dev) == rec["output"]


@pytest.mark.parametrize("r", workloads.CONFIG_RADII[4])
def test_cfg4_full_size_digest_row_sharded(r):
    """Config 4 (8192^2 u16, adaptive mode): one device, and row-sharded over
    2 and 4 'devices' (device 0 listed several times stands in for several
    GPUs: each slab is a separate mtb_filter_host_rows call with its halo
    rows read from the host frame)."""
    px = _frame("cfg4")
    rec = _full(f"cfg4_8192_r{r}_adaptive")
    assert G.sha(px) == rec["input"]
    out, _ = mtb.filter_image(px, 2 * r + 1, mode="adaptive")
    assert G.sha(out.pixels) == rec["output"]
    for k in (2, 4):
        out, _ = mtb.filter_image(px, 2 * r + 1, mode="adaptive", devices=[0] * k)
        assert G.sha(out.pixels) == rec["output"], k


@pytest.mark.parametrize("r", workloads.CONFIG_RADII[5])
def test_cfg5_full_batch_digest(r):
    """Config 5 (64 x 2048^2 u8): the one-launch device batch entry, and the
    host batch spread over 'devices' (plan_images runs through the
    frame-sequence entry) -- every image and the stacked batch equal the
    reference."""
    b5 = _frame("cfg5")
    rec = _full(f"cfg5_batch_r{r}")
    assert G.sha(b5) == rec["input"]
    dev = mtb.rank_filter(torch.from_numpy(b5).cuda(), r).cpu().numpy()
    bad = [i for i in range(64) if G.sha(dev[i]) != _full(f"cfg5_2048_img{i}_r{r}")["output"]]
    assert not bad, bad
    assert G.sha(dev) == rec["output"]
    del dev
    outs = mtb.filter_images(b5, 2 * r + 1, devices=[0] * 3)
    bad = [i for i in range(64) if G.sha(outs[i]) != _full(f"cfg5_2048_img{i}_r{r}")["output"]]
    assert not bad, bad


def _properties(px, out):
    """Size-independent check: every output value occurs in the input."""
    assert out.shape == px.shape and out.dtype == px.dtype
    present = np.zeros(1 << (8 * px.itemsize), dtype=bool)
    present[px.ravel()] = True
    assert present[out.ravel()].all()


def test_full_size_off_centre_ranks():
    """Config-2/3 frames at non-median ranks (no reference digest at full
    size): the outputs occur in the input and are ordered by rank."""
    for key, r in (("cfg2", 15), ("cfg3", 7)):
        px = _frame(key)
        dev = torch.from_numpy(px).cuda()
        n = 2 * r + 1
        prev = None
        for rank in (1, n * n // 4, n * n // 2 + 1, n * n):
            out = mtb.rank_filter(dev, r, rank=rank).cpu().numpy()
            _properties(px, out)
            if prev is not None:
                assert (out >= prev).all(), (key, rank)
            prev = out


# ------------------------------------------ every kernel family vs the oracle

_FAMILY_CASES = [c for c in G.small_cases() if c[0]["rank"] is None and c[0]["percentile"] is None]


@pytest.mark.parametrize("family", ["vert", "ctmf", "bandmma", "bandtc", "sortnet", "colhist", "colhist16s", "colhist16c", "lowsel", "wk16"])
def test_each_kernel_family_is_exact(family, monkeypatch):
    """MTB_KERNEL forces one family; families that do not apply to a case
    (ctmf: 8-bit only; sortnet: median of n <= 7) fall through to the
    default dispatch, so every case must still be exact."""
    from paper_1105_3829_b200 import _lib

    monkeypatch.setenv("MTB_KERNEL", family)
    seen = set()
    for meta, px, ref in _FAMILY_CASES:
        out, _ = mtb.filter_image(mtb.GrayImage(px, meta["bit_depth"]), meta["n"],
                                  **_ref_args(meta))
        assert np.array_equal(out.pixels, ref), (family, meta["idx"])
        seen.add(_lib.last_kernel().split("<")[0])
    rng = np.random.default_rng(7)
    for r in (1, 2, 3, 5, 12, 17, 24, 40, 63):
        px = workloads.cfg2_blur_sp_u8(150, 700 + r)
        out = mtb.rank_filter(torch.from_numpy(px).cuda(), r).cpu().numpy()
        assert np.array_equal(out, O.iot_filter(px, 2 * r + 1)), (family, r)
        seen.add(_lib.last_kernel().split("<")[0])
        px16 = rng.integers(0, 65536, (70, 90)).astype(np.uint16)
        out16 = mtb.rank_filter(torch.from_numpy(px16).cuda(), min(r, 34)).cpu().numpy()
        assert np.array_equal(out16, O.iot_filter(px16, 2 * min(r, 34) + 1)), (family, r)
    expect = {"vert": "k_vert_u8", "ctmf": "k_ctmf_u8", "bandmma": "k_bandmma_u8", "bandtc": "k_bandtc_u8", "sortnet": "k_sortnet", "colhist": "k_colhist_u8",
              "colhist16s": "k_colhist16s_u16", "colhist16c": "k_colhist16c_u16", "lowsel": "k_lowsel_u16",
              "wk16": "k_colhist4p_u8"}[family]
    assert expect in seen, seen


@pytest.mark.parametrize("r", [1, 4, 9, 20, 130])
def test_vert_u16_ranks_and_counter_widths(r, monkeypatch):
    """k_vert_u16 (the general 16-bit path, any radius) on wide-spread and
    compact images at min / max / off-centre ranks, u16 and (r = 130,
    n^2 > 65535) u32 counters."""
    from paper_1105_3829_b200 import _lib

    monkeypatch.setenv("MTB_KERNEL", "vert")
    rng = np.random.default_rng(40 + r)
    h, w = (300, 280) if r == 130 else (90, 110)
    n = 2 * r + 1
    imgs = [rng.integers(0, 65536, (h, w)).astype(np.uint16),
            (30000 + rng.normal(0, 300, (h, w))).clip(0, 65535).astype(np.uint16)]
    for px in imgs:
        for rank in (1, n * n, (n * n) // 3 + 1):
            out = mtb.rank_filter(torch.from_numpy(px).cuda(), r, rank=rank).cpu().numpy()
            assert _lib.last_kernel().startswith("k_vert_u16"), _lib.last_kernel()
            assert np.array_equal(out, O.iot_filter(px, n, rank=rank)), (r, rank)


@pytest.mark.parametrize("var,name", [(0, "k_colhist_u8<128,1>"), (2, "k_colhist_u8<128,2>"),
                                      (12, "k_colhist4_u8<256>"), (13, "k_colhist4_u8<128>"),
                                      (30, "k_colhist4p_u8<256,3>"),
                                      (31, "k_colhist4p_u8<256,2>"), (32, "k_colhist4p_u8<256,4>"),
                                      (34, "k_colhist4p_u8<256,1>")])
def test_colhist_variants_all_group_tails(var, name, monkeypatch):
    """Each column-histogram variant at radii covering every carry-free group
    size G (8/4/2/1) and tail n mod G, ragged tiles (W not a multiple of the
    tile) and min / max / off-centre ranks."""
    from paper_1105_3829_b200 import _lib

    monkeypatch.setenv("MTB_KERNEL", "colhist")
    monkeypatch.setenv("MTB_CH_VAR", str(var))
    rng = np.random.default_rng(90 + var)
    px = workloads.cfg2_blur_sp_u8(160, 601, seed=90 + var)
    noise = rng.integers(0, 256, px.shape).astype(np.uint8)
    for r in (1, 2, 3, 4, 5, 6, 7, 8, 11, 13, 15, 16, 20, 31, 32, 45, 63, 64, 100, 127):
        n = 2 * r + 1
        for img, rank in ((px, None), (noise, 1), (noise, n * n), (px, (n * n) // 5 + 1)):
            out = mtb.rank_filter(torch.from_numpy(img).cuda(), r, rank=rank).cpu().numpy()
            # pair records need 2n <= 255; wider windows fall back to single records
            expect = "k_colhist4_u8<256>" if var >= 30 and 2 * n > 255 else name
            assert _lib.last_kernel() == expect, _lib.last_kernel()
            assert np.array_equal(out, O.iot_filter(img, n, rank=rank)), (var, r, rank)


@pytest.mark.parametrize("wk", ["1", "0"])
@pytest.mark.parametrize("kind", ["compact", "uniform", "two_level"])
def test_colhist16_u16_two_phase(kind, wk, monkeypatch):
    """k_colhist16_u16 (high byte by column records, then one low-byte sweep
    per high byte used by the tile) at radii covering every group size/tail,
    ragged tiles, min / max / off-centre ranks; the uniform image makes many
    high bytes per tile (many low-byte sweeps)."""
    from paper_1105_3829_b200 import _lib

    monkeypatch.setenv("MTB_KERNEL", "colhist")
    monkeypatch.setenv("MTB_CH16_WK", wk)  # window-keyed first sweep on / off
    rng = np.random.default_rng({"compact": 123, "uniform": 321, "two_level": 55}[kind])
    h, w = 150, 300
    if kind == "compact":
        px = (20000 + rng.normal(0, 250, (h, w))).clip(0, 65535).astype(np.uint16)
    elif kind == "two_level":  # tiles straddling the step miss the guessed high byte
        px = (np.where(np.arange(w)[None, :] < 170, 20000, 41000) + rng.normal(0, 200, (h, w)))
        px = px.clip(0, 65535).astype(np.uint16)
    else:
        px = rng.integers(0, 65536, (h, w)).astype(np.uint16)
    for r in (1, 2, 3, 4, 5, 7, 8, 15, 16, 31, 32, 63, 64, 127):
        n = 2 * r + 1
        for rank in (None, 1, n * n, (n * n) // 3 + 1):
            out = mtb.rank_filter(torch.from_numpy(px).cuda(), r, rank=rank).cpu().numpy()
            assert _lib.last_kernel() == "k_colhist16_u16", _lib.last_kernel()
            assert np.array_equal(out, O.iot_filter(px, n, rank=rank)), (kind, r, rank)


def test_colhist16_u16_batch_slab_and_lut(monkeypatch):
    """Two-phase 16-bit kernel through the batch entry (per-image scratch
    planes), a row slab with a pitched output, and a value map."""
    monkeypatch.setenv("MTB_KERNEL", "colhist")
    rng = np.random.default_rng(5)
    imgs = (30000 + rng.normal(0, 400, (3, 90, 130))).clip(0, 65535).astype(np.uint16)
    out = mtb.rank_filter(torch.from_numpy(imgs).cuda(), 6).cpu().numpy()
    for i in range(3):
        assert np.array_equal(out[i], O.iot_filter(imgs[i], 13)), i
    px = imgs[0]
    ref = O.iot_filter(px, 13)
    big = torch.zeros((90, 160), dtype=torch.uint16, device="cuda")
    sl = mtb.rank_filter(torch.from_numpy(px).cuda(), 6, rows=(20, 70), out=big[20:70, :130])
    assert np.array_equal(sl.cpu().numpy(), ref[20:70])
    lut = torch.from_numpy((np.arange(65536) & ~np.uint32(15)).astype(np.uint16)).cuda()
    q = mtb.rank_filter(torch.from_numpy(px).cuda(), 6, lut=lut).cpu().numpy()
    assert np.array_equal(q, ref & ~np.uint16(15))


@pytest.mark.parametrize("family", ["colhist16s", "colhist16c"])
@pytest.mark.parametrize("kind", ["uniform", "compact"])
def test_colhist16_sorted_span_kernels(kind, family, monkeypatch):
    """The sorted-span 16-bit kernels -- k_colhist16s_u16 (column records +
    sorted columns) and k_colhist16c_u16 (pair records + candidate runs,
    with the crowded-bin counting path that compact data takes) -- at radii
    covering every group size/tail, ragged tiles and min / max / off-centre
    ranks; windows past their limits (16s: shared memory at r = 127; 16c:
    pair counts at n > 127) fall back to the two-phase kernel, still exact."""
    from paper_1105_3829_b200 import _lib

    monkeypatch.setenv("MTB_KERNEL", family)
    rng = np.random.default_rng(77 if kind == "compact" else 78)
    h, w = 150, 300
    if kind == "compact":
        px = (20000 + rng.normal(0, 250, (h, w))).clip(0, 65535).astype(np.uint16)
    else:
        px = rng.integers(0, 65536, (h, w)).astype(np.uint16)
    for r in (1, 2, 3, 4, 7, 8, 15, 16, 31, 32, 63, 64, 127):
        n = 2 * r + 1
        for rank in (None, 1, n * n, (n * n) // 3 + 1):
            out = mtb.rank_filter(torch.from_numpy(px).cuda(), r, rank=rank).cpu().numpy()
            fallback = r == 127 if family == "colhist16s" else n > 127
            expect = "k_colhist16_u16" if fallback else f"k_{family}_u16"
            assert _lib.last_kernel() == expect, _lib.last_kernel()
            assert np.array_equal(out, O.iot_filter(px, n, rank=rank)), (kind, r, rank)


def _lowsel_frames(rng, h, w):
    """Spread, compact, mixed (spread with a compact band and a saturated
    corner: blocks whose buckets overflow go to the two-phase kernel) and
    12-bit-in-16 frames."""
    noise = rng.integers(0, 65536, (h, w)).astype(np.uint16)
    compact = (30000 + rng.normal(0, 300, (h, w))).clip(0, 65535).astype(np.uint16)
    mixed = noise.copy()
    mixed[:, w // 3: 2 * w // 3] = compact[:, w // 3: 2 * w // 3]
    mixed[h // 2:, : w // 4] = 65535
    twelve = (rng.integers(0, 4096, (h, w)) * 16).astype(np.uint16)
    return {"noise": noise, "compact": compact, "mixed": mixed, "twelve": twelve}


@pytest.mark.parametrize("ph", ["4", "8", "16"])
@pytest.mark.parametrize("kind", ["noise", "compact", "mixed", "twelve"])
def test_lowsel_u16_candidate_buckets(kind, ph, monkeypatch):
    """The 16-bit candidate-bucket path (high-byte pair records ->
    k_lowsel_u16 -> todo-gated k_colhist16_u16) on ragged frames: radii over
    every column-step count of the scan (2..5) and both pair-record layouts
    of the first pass, min / max / off-centre ranks, frames narrower than a
    block and lower than a block row, the clamped borders (weighted border
    entries) and data whose buckets overflow; block heights 4 and 8 (the
    block's words in registers) and 16 (re-read)."""
    from paper_1105_3829_b200 import _lib

    monkeypatch.setenv("MTB_KERNEL", "lowsel")
    monkeypatch.setenv("MTB_LS_PH", ph)
    rng = np.random.default_rng(123)
    for (h, w) in ((97, 333), (300, 64), (5, 20), (131, 257)):
        px = _lowsel_frames(rng, h, w)[kind]
        src = torch.from_numpy(px).cuda()
        for r in (3, 4, 7, 15, 16, 17, 24, 32, 40, 49, 63):
            n = 2 * r + 1
            if n > 2 * min(h, w) + 1:
                continue
            for rank in (None, 1, n * n, (n * n) // 3 + 1):
                out = mtb.rank_filter(src, r, rank=rank).cpu().numpy()
                assert _lib.last_kernel() == "k_lowsel_u16", _lib.last_kernel()
                assert np.array_equal(out, O.iot_filter(px, n, rank=rank)), (kind, h, w, r, rank)
    # outside its radii the family falls back to the two-phase kernel
    px = _lowsel_frames(rng, 70, 90)[kind]
    for r in (2, 64):
        out = mtb.rank_filter(torch.from_numpy(px).cuda(), r, rank=5).cpu().numpy()
        assert _lib.last_kernel() == "k_colhist16_u16", _lib.last_kernel()
        assert np.array_equal(out, O.iot_filter(px, 2 * r + 1, rank=5)), (kind, r)


@pytest.mark.parametrize("hi", ["pair", "mma"])
def test_lowsel_u16_first_passes_batch_slab_and_lut(hi, monkeypatch):
    """The candidate-bucket path with the first pass forced onto the pair
    records / the band-matrix products at every radius; the batch entry (per-image scratch
    planes and flags), a row slab with a pitched output, a value map, and
    the default device-selected dispatch on a batch that mixes spread and
    compact images."""
    from paper_1105_3829_b200 import _lib

    monkeypatch.setenv("MTB_LS_HI", hi)
    rng = np.random.default_rng(321)
    frames = _lowsel_frames(rng, 120, 200)
    stack = np.stack(list(frames.values()))
    out = mtb.rank_filter(torch.from_numpy(stack).cuda(), 9).cpu().numpy()
    assert "k_lowsel_u16" in _lib.last_kernel(), _lib.last_kernel()
    for i in range(stack.shape[0]):
        assert np.array_equal(out[i], O.iot_filter(stack[i], 19)), i
    monkeypatch.setenv("MTB_KERNEL", "lowsel")
    for r in (6, 31, 50):
        n = 2 * r + 1
        out = mtb.rank_filter(torch.from_numpy(stack).cuda(), r).cpu().numpy()
        for i in range(stack.shape[0]):
            assert np.array_equal(out[i], O.iot_filter(stack[i], n)), (r, i)
        px = frames["mixed"]
        ref = O.iot_filter(px, n)
        big = torch.zeros((120, 240), dtype=torch.uint16, device="cuda")
        sl = mtb.rank_filter(torch.from_numpy(px).cuda(), r, rows=(19, 77), out=big[19:77, :200])
        assert np.array_equal(sl.cpu().numpy(), ref[19:77]), r
        lut = torch.from_numpy((np.arange(65536) & ~np.uint32(15)).astype(np.uint16)).cuda()
        q = mtb.rank_filter(torch.from_numpy(px).cuda(), r, lut=lut).cpu().numpy()
        assert np.array_equal(q, ref & ~np.uint16(15)), r


@pytest.mark.parametrize("bits", [8, 10, 12, 14])
def test_lowsel_u16_key_follows_the_occupied_range(bits):
    """10- / 12-bit noise in 16-bit words looks compact by its high bytes;
    the spread probe then shifts the coarse key to the occupied range
    (key = min(v >> s, 255)) and the candidate-bucket path takes it: host
    entry (probe on the host frame: the kernel is named) and device entry
    (probe on the device), a few outliers above the sampled range (clamped
    into the top key), every rank position."""
    from paper_1105_3829_b200 import _lib

    rng = np.random.default_rng(1000 + bits)
    px = rng.integers(0, 1 << bits, (150, 260)).astype(np.uint16)
    out, _ = mtb.filter_image(px, 11)
    assert _lib.last_kernel() == "k_lowsel_u16", _lib.last_kernel()
    assert np.array_equal(out.pixels, O.iot_filter(px, 11))
    spiky = px.copy()
    spiky[rng.integers(0, 150, 5), rng.integers(0, 260, 5)] = 65535
    for img in (px, spiky):
        src = torch.from_numpy(img).cuda()
        for r in (4, 15, 33):
            n = 2 * r + 1
            for rank in (None, 1, n * n, (n * n) // 3 + 1):
                got = mtb.rank_filter(src, r, rank=rank).cpu().numpy()
                assert np.array_equal(got, O.iot_filter(img, n, rank=rank)), (bits, r, rank)
    # row slabs over "devices" (the host rows entry: halos from the host frame, one probe per slab)
    out, _ = mtb.filter_image(px, 19, devices=[0, 0, 0])
    assert np.array_equal(out.pixels, O.iot_filter(px, 19))
    # peaked data in a narrow range stays on the two-phase kernel (not flat in key space)
    peaked = (800 + rng.normal(0, 40, (150, 260))).clip(0, 65535).astype(np.uint16)
    out, _ = mtb.filter_image(peaked, 11)
    assert _lib.last_kernel() == "k_colhist16_u16", _lib.last_kernel()
    assert np.array_equal(out.pixels, O.iot_filter(peaked, 11))


@pytest.mark.parametrize("kind", ["compact", "drift", "noise", "mixed", "low", "high", "cfg4"])
def test_wk16_window_key_pass(kind, monkeypatch):
    """The window-key pass of compact 16-bit data (k_colhist4p_u8<...,
    uint16_t, 1>: one 8-bit problem per tile around the tile's sampled
    median) with the two-phase kernel on the flagged tiles: data where every
    pixel hits (compact, config 4), where tiles drift away from their window,
    where nothing hits (noise) and windows clamped at 0 and 65535; every rank
    position, a slab, a batch, a value map; and the default dispatch taking
    it for peaked data from r = 40."""
    from paper_1105_3829_b200 import _lib

    rng = np.random.default_rng(77)
    h, w = 131, 333
    noise = rng.integers(0, 65536, (h, w)).astype(np.uint16)
    compact = (30000 + rng.normal(0, 60, (h, w))).clip(0, 65535).astype(np.uint16)
    px = {"compact": compact,
          "drift": (np.add.outer(np.arange(h) * 3, np.arange(w) * 2) + rng.normal(0, 40, (h, w)) + 500).clip(0, 65535).astype(np.uint16),
          "noise": noise,
          "mixed": np.where(np.arange(w)[None, :] < w // 2, compact, noise).astype(np.uint16),
          "low": rng.integers(0, 90, (h, w)).astype(np.uint16),
          "high": (65535 - rng.integers(0, 90, (h, w))).astype(np.uint16),
          "cfg4": workloads.cfg4_three_gauss_u16(h, w)}[kind]
    src = torch.from_numpy(px).cuda()
    if kind in ("compact", "cfg4", "low", "high"):  # peaked: the host entry names the pass
        out, _ = mtb.filter_image(px, 91)
        # ("low": values 0..89 are wide and flat once the key follows the occupied range -> buckets)
        expect = "k_lowsel_u16" if kind == "low" else "k_colhist4p_u8<256,u16 window key>"
        assert _lib.last_kernel() == expect, _lib.last_kernel()
        assert np.array_equal(out.pixels, O.iot_filter(px, 91))
        assert np.array_equal(mtb.rank_filter(src, 45).cpu().numpy(), O.iot_filter(px, 91))
    monkeypatch.setenv("MTB_KERNEL", "wk16")
    for r in (3, 8, 16, 17, 33, 63):
        n = 2 * r + 1
        for rank in (None, 1, n * n, (n * n) // 3 + 1):
            out = mtb.rank_filter(src, r, rank=rank).cpu().numpy()
            assert _lib.last_kernel() == "k_colhist4p_u8<256,u16 window key>", _lib.last_kernel()
            assert np.array_equal(out, O.iot_filter(px, n, rank=rank)), (kind, r, rank)
    ref = O.iot_filter(px, 13)
    big = torch.zeros((h, 400), dtype=torch.uint16, device="cuda")
    sl = mtb.rank_filter(src, 6, rows=(19, 77), out=big[19:77, :w])
    assert np.array_equal(sl.cpu().numpy(), ref[19:77])
    lut = torch.from_numpy((np.arange(65536) & ~np.uint32(15)).astype(np.uint16)).cuda()
    assert np.array_equal(mtb.rank_filter(src, 6, lut=lut).cpu().numpy(), ref & ~np.uint16(15))
    stack = np.stack([px, px[::-1].copy(), noise])
    got = mtb.rank_filter(torch.from_numpy(stack).cuda(), 6).cpu().numpy()
    for i in range(3):
        assert np.array_equal(got[i], O.iot_filter(stack[i], 13)), i


# ------------------------------------------ 3x3 kernels (k_med3_u8 / k_med3t_u8)

def _pitched(px, pad):
    """CUDA view of px whose rows sit in a buffer `pad` columns wider than
    the next multiple of 16 (aligned pitch, as the vector / TMA paths need)."""
    H, W = px.shape
    buf = torch.zeros((H, ((W + 15) & ~15) + pad), dtype=torch.from_numpy(px).dtype, device="cuda")
    buf[:, :W] = torch.from_numpy(px).cuda()
    return buf[:, :W]


@pytest.mark.parametrize("tma,rt", [("1", "1"), ("1", "2"), ("1", "8"), ("1", "40"),
                                    ("0", "1"), ("0", "2"), ("0", "8"), ("0", "32")])
def test_med3_u8_shapes_slabs_batch_lut(tma, rt, monkeypatch):
    """3x3 median, both kernels (TMA-staged for W % 16 == 0 with aligned
    rows, register-resident otherwise): every width tail (partial last lane
    and CTA, widths below one lane), odd and even band heights, slab calls,
    batch, value map, unaligned pitches.  All vs the oracle."""
    from paper_1105_3829_b200 import _lib

    monkeypatch.setenv("MTB_MED3T", tma)
    monkeypatch.setenv("MTB_MED3_MIN_RT", rt)
    rng = np.random.default_rng(31)

    def expect(W, aligned=True):
        return "k_med3t_u8" if (tma == "1" and W % 16 == 0 and aligned) else "k_med3_u8"

    for H, W in [(1, 1), (1, 9), (2, 3), (3, 8), (5, 7), (1, 16), (2, 32), (17, 255), (19, 256),
                 (33, 257), (40, 1023), (35, 1025), (21, 1040), (300, 1040), (21, 2100), (64, 64),
                 (9, 4096)]:
        px = rng.integers(0, 256, (H, W), dtype=np.uint8)
        ref = O.iot_filter(px, 3)
        for pad in (0, 8):
            o = _pitched(np.zeros_like(px), pad)
            out = mtb.rank_filter(_pitched(px, pad), 1, out=o).cpu().numpy()
            assert _lib.last_kernel() == expect(W, pad == 0), (H, W, pad, _lib.last_kernel())
            assert np.array_equal(out, ref), (H, W, pad)
    # slabs of a frame, each with its 1-row halo
    for W in (300, 320):
        px = workloads.cfg2_blur_sp_u8(61, W)
        ref = O.iot_filter(px, 3)
        dev = _pitched(px, 0)
        for a, b in [(0, 7), (7, 30), (30, 61), (60, 61)]:
            s0, s1 = max(a - 1, 0), min(b + 1, 61)
            o = _pitched(np.zeros((b - a, W), np.uint8), 0)
            out = mtb.rank_filter(dev[s0:s1], 1, out=o, rows=(a, b), src_row0=s0, height=61)
            assert _lib.last_kernel() == expect(W)
            assert np.array_equal(out.cpu().numpy(), ref[a:b]), (W, a, b)
    # batch
    for W in (136, 144):
        b5 = workloads.cfg5_batch_u8(3, 70, W)
        out = mtb.rank_filter(torch.from_numpy(b5).cuda(), 1).cpu().numpy()
        assert _lib.last_kernel() == expect(W)
        for i in range(3):
            assert np.array_equal(out[i], O.iot_filter(b5[i], 3)), (W, i)
    # reduced precision through the value map
    for W in (333, 336):
        px = rng.integers(0, 256, (45, W), dtype=np.uint8)
        o, _ = mtb.filter_image(px, 3, max_error=16)
        assert np.array_equal(o.pixels, O.iot_filter(px, 3, max_error=16)), W
    # unaligned pitches (byte loads / stores), and the forced selection network
    for W in (101, 1029, 2050):
        px = rng.integers(0, 256, (30, W), dtype=np.uint8)
        out = mtb.rank_filter(torch.from_numpy(px).cuda(), 1).cpu().numpy()
        assert _lib.last_kernel() == "k_med3_u8"
        assert np.array_equal(out, O.iot_filter(px, 3)), W
    monkeypatch.setenv("MTB_KERNEL", "sortnet")
    out = mtb.rank_filter(torch.from_numpy(px).cuda(), 1).cpu().numpy()
    assert _lib.last_kernel() == "k_sortnet<3>"
    assert np.array_equal(out, O.iot_filter(px, 3))


# ------------------------------------------ n = 5, 7 medians (k_mednet)

@pytest.mark.parametrize("bits", [8, 16])
@pytest.mark.parametrize("rt", ["2", "16", "40"])
def test_mednet_shapes_slabs_batch_lut(bits, rt, monkeypatch):
    """k_mednet (sorted packed columns, shared merges): n = 5 and 7, 8- and
    16-bit, widths around the 512-column CTA tile and the 4-column thread
    tile, heights 1..RT+3 (odd band tails), slabs, batch, value map, ties
    (few distinct values).  All vs the oracle."""
    from paper_1105_3829_b200 import _lib

    monkeypatch.setenv("MTB_KERNEL", "mednet")
    monkeypatch.setenv("MTB_MN_MIN_RT", rt)
    rng = np.random.default_rng(57 + bits)
    hi = 256 if bits == 8 else 65536
    dt = np.uint8 if bits == 8 else np.uint16
    for n in (5, 7):
        for H, W in [(1, 1), (2, 5), (3, 3), (7, 7), (5, 13), (9, 512), (17, 513), (33, 1030),
                     (41, 300), (64, 64), (20, 2053)]:
            if n > 2 * min(H, W) + 1:
                continue
            for vals in (hi, 3):
                px = rng.integers(0, vals, (H, W)).astype(dt)
                out = mtb.rank_filter(torch.from_numpy(px).cuda(), n // 2).cpu().numpy()
                assert _lib.last_kernel().startswith("k_mednet"), _lib.last_kernel()
                assert np.array_equal(out, O.iot_filter(px, n)), (n, H, W, vals)
        # slabs of a 61-row frame with their halos
        px = rng.integers(0, hi, (61, 700)).astype(dt)
        ref = O.iot_filter(px, n)
        r = n // 2
        dev = torch.from_numpy(px).cuda()
        for a, b in [(0, 9), (9, 30), (30, 61), (60, 61)]:
            s0, s1 = max(a - r, 0), min(b + r, 61)
            out = mtb.rank_filter(dev[s0:s1], r, rows=(a, b), src_row0=s0, height=61)
            assert np.array_equal(out.cpu().numpy(), ref[a:b]), (n, a, b)
        # batch
        bt = rng.integers(0, hi, (3, 40, 520)).astype(dt)
        out = mtb.rank_filter(torch.from_numpy(bt).cuda(), r).cpu().numpy()
        for i in range(3):
            assert np.array_equal(out[i], O.iot_filter(bt[i], n)), (n, i)
        # value map (reduced precision)
        o, _ = mtb.filter_image(px, n, max_error=16)
        assert np.array_equal(o.pixels, O.iot_filter(px, n, max_error=16)), n


_SERIAL_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_1105_3829_b200 as mtb, workloads
from oracle import oracle as O
torch.cuda.set_device(0)
px = workloads.cfg2_blur_sp_u8(700, 900)
pin = torch.from_numpy(px).pin_memory().numpy()
for r in (7, 15, 31):
    ref = O.iot_filter(px, 2 * r + 1)
    out, _ = mtb.filter_image(px, 2 * r + 1)
    assert np.array_equal(out.pixels, ref), ("pageable", r)
    assert np.array_equal(mtb.filter_host_buffer(pin, r), ref), ("pinned", r)
    outs = mtb.filter_host_frames([pin, px], [r, r + 1])
    assert np.array_equal(outs[0], ref), ("frames", r)
px16 = workloads.cfg4_three_gauss_u16(600, 500)
out, _ = mtb.filter_image(torch.from_numpy(px16).pin_memory().numpy(), 31)
assert np.array_equal(out.pixels, O.iot_filter(px16, 31))
print("SERIAL_OK")
"""


def test_host_paths_under_serialised_launches():
    """CUDA_LAUNCH_BLOCKING=1 serialises every launch (as profilers and
    sanitizers do): the streaming host paths enqueue all their copies and
    row-arrival writes before the kernel whose CTAs wait on them, so they
    must still finish (r = 15, 31: the streaming launch) and be exact."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CUDA_LAUNCH_BLOCKING="1")
    res = subprocess.run([sys.executable, "-c", _SERIAL_SCRIPT.format(root=root)], env=env,
                         capture_output=True, text=True, timeout=300)
    assert res.returncode == 0 and "SERIAL_OK" in res.stdout, res.stdout[-2000:] + res.stderr[-4000:]


def test_filter_images_over_devices():
    """filter_images: a batch spread over 'devices' (device 0 listed several
    times stands in for several GPUs), mixed 8-bit content, ranks and a
    value map; every image equal to its own filter_image result / oracle."""
    b = workloads.cfg5_batch_u8(7, 150, 140)
    for devs in ([0], [0, 0], [0, 0, 0, 0]):
        outs = mtb.filter_images(b, 15, devices=devs)
        for i in range(b.shape[0]):
            assert np.array_equal(outs[i], O.iot_filter(b[i], 15)), (devs, i)
    outs = mtb.filter_images(list(b[:3]), 9, rank=5, devices=[0, 0])
    for i in range(3):
        assert np.array_equal(outs[i], O.iot_filter(b[i], 9, rank=5))
    outs = mtb.filter_images(b[:4], 5, max_error=16, devices=[0, 0])
    for i in range(4):
        assert np.array_equal(outs[i], O.iot_filter(b[i], 5, max_error=16))
    with pytest.raises(ValueError):
        mtb.filter_images([b[0], b[0][:10]], 5)
    assert mtb.filter_images([], 5) == []


def test_rank_filter_checks_out_and_device():
    """rank_filter rejects an `out` of the wrong dtype, device or shape
    instead of writing out of bounds."""
    px = torch.from_numpy(np.arange(64 * 80, dtype=np.uint16).reshape(64, 80).copy()).cuda()
    with pytest.raises(ValueError):
        mtb.rank_filter(px, 2, out=torch.empty((64, 80), dtype=torch.uint8, device="cuda"))
    with pytest.raises(ValueError):
        mtb.rank_filter(px, 2, out=torch.empty((64, 80), dtype=torch.uint16))
    with pytest.raises(ValueError):
        mtb.rank_filter(px, 2, out=torch.empty((60, 80), dtype=torch.uint16, device="cuda"))
    b = px.reshape(4, 16, 80)
    with pytest.raises(ValueError):
        mtb.rank_filter(b, 2, out=torch.empty((4, 16, 79), dtype=torch.uint16, device="cuda"))
    with pytest.raises(ValueError):
        mtb.filter_host_buffer(px.cpu().numpy(), 2, lut=np.arange(256, dtype=np.uint16))
    s = torch.cuda.Stream()
    out = mtb.rank_filter(px, 2, stream=s)
    s.synchronize()
    assert np.array_equal(out.cpu().numpy(), O.iot_filter(px.cpu().numpy(), 5))


@pytest.mark.parametrize("ndev", [2, 3])
def test_filter_image_device_slabs(ndev):
    """filter_image(devices=[...]): one row slab per listed device with its
    halo rows from the host copy (the multi-GPU decomposition; the same
    device listed several times stands in for several GPUs here) -- equal to
    the single-device result and the oracle, 8- and 16-bit, with bands."""
    rng = np.random.default_rng(ndev)
    px = workloads.cfg2_blur_sp_u8(301, 257, seed=ndev)
    for n in (3, 9, 31):
        out, _ = mtb.filter_image(px, n, devices=[0] * ndev, bands=2)
        assert np.array_equal(out.pixels, O.iot_filter(px, n)), n
    px16 = rng.integers(0, 65536, (123, 80)).astype(np.uint16)
    out = mtb.median_filter(px16, 4, devices=[0] * ndev)
    assert np.array_equal(out, O.iot_filter(px16, 9))


@pytest.mark.parametrize("pre,ctb4", [("1", "1000"), ("1", "1"), ("0", "1000")])
def test_ctmf_slabs_batch_lut(pre, ctb4, monkeypatch):
    """The CTMF tile kernel with up-front span snapshots (both register
    budgets) and with per-tile scans: slab calls with row_begin > 0 (the
    snapshot rows follow the slab), a batch of images (one snapshot set per
    image), a value map, a ragged last tile column -- all vs the oracle."""
    from paper_1105_3829_b200 import _lib

    monkeypatch.setenv("MTB_KERNEL", "ctmf")
    monkeypatch.setenv("MTB_CT_PRE", pre)
    monkeypatch.setenv("MTB_CT_CTB4_R", ctb4)
    px = workloads.cfg2_blur_sp_u8(230, 333, seed=11)
    H = px.shape[0]
    for r in (33, 48, 63):
        ref = O.iot_filter(px, 2 * r + 1)
        dev = torch.from_numpy(px).cuda()
        for a, b in [(0, 57), (57, 170), (170, 230)]:
            top, bot = max(0, a - r), min(H, b + r)
            out = mtb.rank_filter(dev[top:bot], r, rows=(a, b), src_row0=top, height=H)
            assert _lib.last_kernel().startswith("k_ctmf_u8")
            assert np.array_equal(out.cpu().numpy(), ref[a:b]), (r, a, b)
    bt = workloads.cfg5_batch_u8(3, 150, 290)
    out = mtb.rank_filter(torch.from_numpy(bt).cuda(), 40).cpu().numpy()
    for i in range(3):
        assert np.array_equal(out[i], O.iot_filter(bt[i], 81)), i
    o, _ = mtb.filter_image(px, 99, max_error=8)
    assert np.array_equal(o.pixels, O.iot_filter(px, 99, max_error=8))


@pytest.mark.parametrize("tw", ["512", "208", "64"])
def test_bandmma_slabs_batch_lut_ranks(tw, monkeypatch):
    """The band-matrix tensor-core kernel (k_bandmma_u8) at several stripe
    widths: every k-tile count (r = 1 .. 127), ranks at both ends and off
    centre, slab calls with row_begin > 0, a batch of images, a value map,
    ragged stripes -- on smooth frames (keyed windows predicted from the row
    above hit) and on frames whose medians jump between rows and columns
    (every prediction misses: the coarse fallback resolves them) -- all vs the
    oracle."""
    from paper_1105_3829_b200 import _lib

    monkeypatch.setenv("MTB_KERNEL", "bandmma")
    monkeypatch.setenv("MTB_BM_TW", tw)
    rng = np.random.default_rng(int(tw))
    smooth = workloads.cfg2_blur_sp_u8(140, 333, seed=12)
    noise = rng.integers(0, 256, (140, 333), dtype=np.uint8)
    # bands of very different levels, 9 rows / 21 columns wide: the median jumps
    jumpy = ((np.arange(140)[:, None] // 9 * 83 + np.arange(333)[None, :] // 21 * 57) % 256).astype(np.uint8)
    jumpy[rng.random(jumpy.shape) < 0.1] = 255
    for name, px in (("smooth", smooth), ("noise", noise), ("jumpy", jumpy)):
        dev = torch.from_numpy(px).cuda()
        for r in (1, 8, 9, 24, 25, 40, 41, 56, 57, 63, 69):
            n = 2 * r + 1
            for rank in (None, 1, n * n, (n * n) // 3 + 1):
                out = mtb.rank_filter(dev, r, rank=rank).cpu().numpy()
                assert _lib.last_kernel().startswith("k_bandmma_u8"), _lib.last_kernel()
                assert np.array_equal(out, O.iot_filter(px, n, rank=rank)), (name, r, rank)
    tall = workloads.cfg2_blur_sp_u8(300, 150, seed=13)
    for r in (73, 88, 89, 104, 105, 120, 127):  # k-tile counts 6 .. 9
        out = mtb.rank_filter(torch.from_numpy(tall).cuda(), r).cpu().numpy()
        assert np.array_equal(out, O.iot_filter(tall, 2 * r + 1)), r
    H = smooth.shape[0]
    ref = O.iot_filter(smooth, 81)
    dev = torch.from_numpy(smooth).cuda()
    for a, b in [(0, 57), (57, 130), (130, 140)]:
        top, bot = max(0, a - 40), min(H, b + 40)
        out = mtb.rank_filter(dev[top:bot], 40, rows=(a, b), src_row0=top, height=H)
        assert np.array_equal(out.cpu().numpy(), ref[a:b]), (a, b)
    bt = workloads.cfg5_batch_u8(3, 150, 290)
    out = mtb.rank_filter(torch.from_numpy(bt).cuda(), 33).cpu().numpy()
    for i in range(3):
        assert np.array_equal(out[i], O.iot_filter(bt[i], 67)), i
    o, _ = mtb.filter_image(smooth, 99, max_error=8)
    assert np.array_equal(o.pixels, O.iot_filter(smooth, 99, max_error=8))


@pytest.mark.parametrize("tiles,nf", [("4", "32"), ("2", "64"), ("1", "32")])
def test_bandtc_slabs_batch_lut_ranks(tiles, nf, monkeypatch):
    """The tcgen05 band-matrix kernel (k_bandtc_u8: band tiles in tensor
    memory, planes through shared-memory matrix descriptors, accumulators
    read back per pixel) with 1, 2 and 4 tiles of 128 pixels per CTA and both
    window widths: small and large radii, ranks at both ends and off centre,
    slabs, a batch, a value map, ragged stripes, smooth frames (the window
    predicted from the row above holds) and frames whose medians jump (the
    retry from the missed side resolves them), the streaming host entry --
    all vs the oracle."""
    from paper_1105_3829_b200 import _lib

    monkeypatch.setenv("MTB_KERNEL", "bandtc")
    monkeypatch.setenv("MTB_BT_TILES", tiles)
    monkeypatch.setenv("MTB_BT_NF", nf)
    rng = np.random.default_rng(int(tiles) * 100 + int(nf))
    smooth = workloads.cfg2_blur_sp_u8(140, 333, seed=14)
    noise = rng.integers(0, 256, (140, 333), dtype=np.uint8)
    jumpy = ((np.arange(140)[:, None] // 9 * 83 + np.arange(333)[None, :] // 21 * 57) % 256).astype(np.uint8)
    jumpy[rng.random(jumpy.shape) < 0.1] = 255
    flat = np.full((140, 333), 255, dtype=np.uint8)  # the top bin
    flat[::7, ::5] = 0
    for name, px in (("smooth", smooth), ("noise", noise), ("jumpy", jumpy), ("flat", flat)):
        dev = torch.from_numpy(px).cuda()
        for r in (1, 9, 31, 48, 63, 69):
            n = 2 * r + 1
            for rank in (None, 1, n * n, (n * n) // 3 + 1):
                out = mtb.rank_filter(dev, r, rank=rank).cpu().numpy()
                assert _lib.last_kernel().startswith("k_bandtc_u8"), _lib.last_kernel()
                assert np.array_equal(out, O.iot_filter(px, n, rank=rank)), (name, r, rank)
    tall = workloads.cfg2_blur_sp_u8(300, 150, seed=15)
    for r in (76, 97, 112, 127):
        out = mtb.rank_filter(torch.from_numpy(tall).cuda(), r).cpu().numpy()
        assert np.array_equal(out, O.iot_filter(tall, 2 * r + 1)), r
    H = smooth.shape[0]
    ref = O.iot_filter(smooth, 81)
    dev = torch.from_numpy(smooth).cuda()
    for a, b in [(0, 57), (57, 130), (130, 140)]:
        top, bot = max(0, a - 40), min(H, b + 40)
        out = mtb.rank_filter(dev[top:bot], 40, rows=(a, b), src_row0=top, height=H)
        assert np.array_equal(out.cpu().numpy(), ref[a:b]), (a, b)
    bt = workloads.cfg5_batch_u8(3, 150, 290)
    out = mtb.rank_filter(torch.from_numpy(bt).cuda(), 33).cpu().numpy()
    for i in range(3):
        assert np.array_equal(out[i], O.iot_filter(bt[i], 67)), i
    o, _ = mtb.filter_image(smooth, 99, max_error=8)
    assert np.array_equal(o.pixels, O.iot_filter(smooth, 99, max_error=8))
    big = workloads.cfg2_blur_sp_u8(700, 900, seed=16)
    pinned = torch.from_numpy(big).pin_memory()
    got = mtb.filter_host_buffer(pinned.numpy(), 80)  # page-locked source, r >= 12: the streaming launch
    assert np.array_equal(got, O.iot_filter(big, 161))


# ------------------------------------------ every radius through the default dispatch

_SWEEP_R = list(range(1, 71)) + [80, 90, 97]  # 97: the largest window a 97-row frame allows


@pytest.mark.parametrize("kind", ["u8", "u8_smooth", "u16_uniform", "u16_compact"])
def test_default_dispatch_every_radius(kind):
    """Each radius 1..70 (and a spread above) through the default dispatch on
    a ragged 97 x 333 frame: every compile-time window side the kernels are
    instantiated for (merge networks, 16-bin, radix-4 and pair-record
    column histograms, the sorted-column and two-phase 16-bit kernels, the
    CTMF tiles) meets the oracle, for the median and an off-centre rank."""
    from paper_1105_3829_b200 import _lib

    rng = np.random.default_rng({"u8": 91, "u8_smooth": 94, "u16_uniform": 92, "u16_compact": 93}[kind])
    h, w = 97, 333
    if kind == "u8":
        px = rng.integers(0, 256, (h, w)).astype(np.uint8)
    elif kind == "u8_smooth":  # few levels, long runs: many rows whose in/out pixels cancel
        px = ((np.arange(w)[None, :] // 40 + np.arange(h)[:, None] // 30) * 37 % 256
              + rng.integers(0, 2, (h, w))).astype(np.uint8)
    elif kind == "u16_uniform":
        px = rng.integers(0, 65536, (h, w)).astype(np.uint16)
    else:
        px = (30000 + rng.normal(0, 300, (h, w))).clip(0, 65535).astype(np.uint16)
    dev = torch.from_numpy(px).cuda()
    seen = set()
    for r in _SWEEP_R:
        n = 2 * r + 1
        for rank in (None, (n * n) // 5 + 1):
            out = mtb.rank_filter(dev, r, rank=rank).cpu().numpy()
            seen.add(_lib.last_kernel())
            assert np.array_equal(out, O.iot_filter(px, n, rank=rank)), (kind, r, rank, _lib.last_kernel())
    assert len(seen) >= 3, seen
    with pytest.raises(ValueError):
        mtb.rank_filter(dev, 98)
