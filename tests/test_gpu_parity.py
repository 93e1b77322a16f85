"""GPU parity: the CUDA path (through the C ABI) against the reference's own
outputs (golden fixtures) and against the float64 oracle on seeded
config-like inputs; size-independent properties at larger sizes."""

import numpy as np
import pytest

import oracle
from paper_1009_0958_b200 import _lib
from paper_1009_0958_b200 import (
    REFLECT, REPLICATE, RasterImage, apply_filter, filter_batch_device, filter_device,
    filter_host, filter_rows_device, last_fixup_count, parse_filter_spec, synth,
)

pytestmark = pytest.mark.gpu


def _policy(name):
    return REPLICATE if name == "replicate" else REFLECT


def test_golden_cases_bit_exact(cuda, golden):
    data, cases = golden
    bad = []
    for i, c in enumerate(cases):
        img = RasterImage(data[f"in{i}"].astype(np.float64))
        out = apply_filter(img, parse_filter_spec(c["spec"]), _policy(c["border"]))
        if not (out.pixels == data[f"out{i}"]).all():
            bad.append((i, c, int((out.pixels != data[f"out{i}"]).any(-1).sum())))
    assert not bad, bad[:10]


def test_acceptance_criterion4_bit_exact(cuda, golden):
    data, _ = golden
    torch = cuda
    x = torch.from_numpy(data["acc_in"]).cuda()
    for spec in ("vmf", "bvdf:exact", "ddf:exact", "acwddf:exact"):
        got = filter_batch_device(x, parse_filter_spec(spec)).cpu().numpy()
        assert (got == data["acc_out_" + spec.replace(":", "_")]).all(), spec


SPECS = [
    "vmf", "vmf:p=1", "vmf:p=3", "bvdf:exact", "bvdf:minimax", "bvdf:minimax:q=2", "bvdf:minimax:q=3",
    "bvdf:rgb", "bvdf:rgb:p=1", "ddf:exact", "ddf:minimax", "ddf:rgb", "ddf:exact:p=1",
    "acwddf:exact", "acwddf:minimax", "acwddf:rgb", "acwddf:exact:lambda=3:T=5",
    "bvdf:exact:window=5", "bvdf:minimax:window=5", "bvdf:rgb:window=5", "ddf:exact:window=5",
    "ddf:minimax:window=5", "ddf:rgb:window=5", "acwddf:exact:window=5", "acwddf:minimax:window=5",
    "acwddf:rgb:window=5", "vmf:window=5", "ddf:exact:window=7", "bvdf:exact:window=7",
    "bvdf:minimax:window=7", "ddf:rgb:window=7", "acwddf:exact:window=7", "vmf:window=7",
]


def _mismatch_report(got, want, diag):
    bad = (got != want).any(-1)
    nb = int(bad.sum())
    gaps = diag["gap"][bad]
    tm = diag["tmargin"][bad]
    return nb, gaps, tm


@pytest.mark.parametrize("spec", SPECS)
@pytest.mark.parametrize("border", ["replicate", "reflect"])
def test_against_oracle_config_like(cuda, spec, border):
    """Seeded gradient+rectangles+noise images (SURVEY 8(d) generator), odd
    sizes to exercise partial tiles; bit-exact against the float64 oracle."""
    torch = cuda
    s = parse_filter_spec(spec)
    H, W = (150, 173) if s.window < 7 else (77, 101)
    for seed, noise in ((11, ("uncorrelated", 0.15)), (12, ("correlated", 0.20))):
        img = synth.noisy_image(H, W, seed, noise)
        want = oracle.filter_image(img, s, border, diag=True)
        got = filter_device(torch.from_numpy(img).cuda(), s, _policy(border)).cpu().numpy()
        nb, gaps, tm = _mismatch_report(got, want["out"], want)
        assert nb == 0, f"{spec} {border} seed {seed}: {nb} mismatches, gaps {gaps[:8]}, tmargins {tm[:8]}"


@pytest.mark.parametrize("spec", ["bvdf:exact", "ddf:exact", "ddf:minimax:window=5", "acwddf:rgb:window=5"])
def test_uniform_random_images(cuda, spec):
    """Uniform random pixels cover the whole cosine domain (reference's
    random_image, T/_synth.py:56-59)."""
    torch = cuda
    rng = np.random.default_rng(20240)
    img = rng.integers(0, 256, (96, 130, 3)).astype(np.uint8)
    s = parse_filter_spec(spec)
    want = oracle.filter_image(img, s)
    got = filter_device(torch.from_numpy(img).cuda(), s).cpu().numpy()
    assert (got == want).all()


def test_workers_and_rows_bit_identical(cuda):
    """Row partitions (reference workers > 1, filters.py:416-430) and strips
    with halos give the same pixels as the whole-image call."""
    torch = cuda
    img = synth.noisy_image(203, 97, 21, ("correlated", 0.2))
    for spec in ("vmf", "bvdf:minimax", "acwddf:exact", "ddf:exact:window=7"):
        s = parse_filter_spec(spec)
        full = apply_filter(RasterImage(img.astype(np.float64)), s)
        part = apply_filter(RasterImage(img.astype(np.float64)), s, workers=5)
        assert full == part, spec
        # a strip with its halo only
        h = s.window // 2
        x = torch.from_numpy(img).cuda()
        r0, r1 = 50, 131
        strip = x[r0 - h:r1 + h]
        got = filter_rows_device(strip, img.shape[0], r0 - h, r0, r1 - r0, s).cpu().numpy()
        assert (got == full.pixels[r0:r1]).all(), spec


def test_batch_equals_frames(cuda):
    torch = cuda
    frames = np.stack([synth.noisy_image(45, 70, 1000 + i, ("uncorrelated", 0.1)) for i in range(5)])
    s = parse_filter_spec("acwddf:exact")
    got = filter_batch_device(torch.from_numpy(frames).cuda(), s).cpu().numpy()
    for i in range(5):
        want = filter_device(torch.from_numpy(frames[i]).cuda(), s).cpu().numpy()
        assert (got[i] == want).all()


def test_host_path_equals_device_path(cuda):
    torch = cuda
    img = synth.noisy_image(130, 257, 2, ("uncorrelated", 0.15))
    s = parse_filter_spec("ddf:exact")
    a = filter_host(img, s)
    b = filter_device(torch.from_numpy(img).cuda(), s).cpu().numpy()
    assert (a == b).all()


def test_properties_at_config_size(cuda):
    """At a BASELINE-size frame (C2: 1024^2 DDF 3x3 exact): selection
    property (each output is a pixel of its window), determinism, and the
    re-decision rate stays small."""
    torch = cuda
    img = synth.config_input("c2")
    s = parse_filter_spec("ddf:exact")
    x = torch.from_numpy(img).cuda()
    last_fixup_count()  # reset
    a = filter_device(x, s)
    nfix = last_fixup_count()
    b = filter_device(x, s)
    assert torch.equal(a, b)
    out = a.cpu().numpy()
    pad = np.pad(img, ((1, 1), (1, 1), (0, 0)), mode="edge")
    member = np.zeros(img.shape[:2], bool)
    for u in range(3):
        for v in range(3):
            member |= (pad[u:u + img.shape[0], v:v + img.shape[1]] == out).all(-1)
    assert member.all()
    assert nfix < 0.005 * img.shape[0] * img.shape[1], nfix


def test_constant_image_fixed_point_and_idempotence(cuda):
    img = RasterImage(np.full((37, 41, 3), 31.0))
    for spec in ("vmf", "bvdf:minimax", "ddf:rgb", "acwddf:exact", "ddf:minimax:window=7"):
        out = img
        for _ in range(2):
            out = apply_filter(out, parse_filter_spec(spec))
        assert out == img


def test_invalid_inputs_raise(cuda):
    with pytest.raises(ValueError):
        apply_filter(RasterImage(np.full((4, 4, 3), 0.5)), parse_filter_spec("vmf"))
    with pytest.raises(ValueError):
        apply_filter(RasterImage(np.full((4, 4, 3), 256.0)), parse_filter_spec("vmf"))
    with pytest.raises(NotImplementedError):
        apply_filter(RasterImage(np.full((4, 4, 3), 5.0)), parse_filter_spec("vmf:window=33"))


@pytest.mark.parametrize("spec,border", [("ddf:exact:window=7", "reflect"), ("acwddf:minimax:window=5", "replicate"),
                                         ("bvdf:rgb", "reflect")])
def test_host_pipeline_bands(cuda, spec, border):
    """dfg_filter_host pipelines H2D / kernel / D2H over row bands; bands
    must reproduce the whole-image device call exactly."""
    torch = cuda
    img = synth.noisy_image(1100, 190, 5, ("correlated", 0.2))
    s = parse_filter_spec(spec)
    pin = torch.from_numpy(img).pin_memory()
    out = torch.empty_like(pin).pin_memory()
    a = filter_host(pin.numpy(), s, _policy(border), out=out.numpy())
    b = filter_device(torch.from_numpy(img).cuda(), s, _policy(border)).cpu().numpy()
    assert (a == b).all()


S3_SPECS = ["vmf", "vmf:p=3", "bvdf:exact", "bvdf:minimax:q=3", "bvdf:rgb", "bvdf:rgb:p=1", "ddf:exact", "ddf:minimax",
            "ddf:rgb", "ddf:exact:p=1", "acwddf:exact", "acwddf:minimax", "acwddf:rgb", "acwddf:exact:lambda=1:T=3"]


@pytest.mark.parametrize("kernel", ["w3", "cta"])
@pytest.mark.parametrize("spec", S3_SPECS)
def test_3x3_kernels_against_oracle(cuda, spec, kernel):
    """Both 3x3 schedules (warp row-sweep and CTA tiles) are bit-exact,
    including strips, frames, partial last chunks and both borders."""
    with _lib.option("s3_schedule", 1 if kernel == "w3" else 2):
        _check_3x3(cuda, spec)


def _check_3x3(torch, spec):
    s = parse_filter_spec(spec)
    for H, W, seed, border in ((97, 61, 3, "replicate"), (40, 29, 4, "reflect"), (133, 90, 5, "replicate")):
        img = synth.noisy_image(H, W, seed, ("correlated", 0.2))
        img[5:9, 7:12] = 0  # zero vectors (raw 0 vs gray-mapped 1)
        want = oracle.filter_image(img, s, border)
        got = filter_device(torch.from_numpy(img).cuda(), s, _policy(border)).cpu().numpy()
        assert (got == want).all(), (spec, kernel, H, W, int((got != want).any(-1).sum()))
    frames = np.stack([synth.noisy_image(33, 45, 70 + i, ("uncorrelated", 0.15)) for i in range(3)])
    got = filter_batch_device(torch.from_numpy(frames).cuda(), s).cpu().numpy()
    for i in range(3):
        assert (got[i] == oracle.filter_image(frames[i], s)).all()
    img = synth.noisy_image(120, 77, 8, ("uncorrelated", 0.15))
    full = oracle.filter_image(img, s)
    x = torch.from_numpy(img).cuda()
    got = filter_rows_device(x[30:91], 120, 30, 31, 59, s).cpu().numpy()
    assert (got == full[31:90]).all()


@pytest.mark.parametrize("spec", ["ddf:exact", "bvdf:minimax:q=3", "acwddf:rgb", "vmf", "ddf:exact:p=1"])
def test_host_pinned_odd_offsets_3x3_against_oracle(cuda, spec):
    """3x3 through the host pipeline with pinned host buffers at odd byte
    offsets, widths whose rows are not 4-byte multiples, single-row /
    single-column images, both borders and zero vectors: the oracle bit for
    bit, and no stray writes around the output buffer."""
    torch = cuda
    s = parse_filter_spec(spec)
    for H, W, seed, border, shift in ((97, 61, 3, "replicate", 0), (40, 29, 4, "reflect", 1), (133, 90, 5, "replicate", 3),
                                      (1, 37, 6, "replicate", 2), (23, 1, 7, "reflect", 1), (64, 31, 8, "reflect", 0)):
        img = synth.noisy_image(H, W, seed, ("correlated", 0.2))
        if H > 9 and W > 12:
            img[5:9, 7:12] = 0
        n = img.size
        buf_in = torch.zeros(n + 8, dtype=torch.uint8).pin_memory()
        buf_out = torch.full((n + 8,), 7, dtype=torch.uint8).pin_memory()
        a_in = buf_in.numpy()[shift:shift + n].reshape(img.shape)
        a_out = buf_out.numpy()[3 - shift:3 - shift + n].reshape(img.shape)
        a_in[...] = img
        got = filter_host(a_in, s, _policy(border), out=a_out)
        want = oracle.filter_image(img, s, border)
        assert (got == want).all(), (spec, H, W, border, int((got != want).any(-1).sum()))
        guard = buf_out.numpy()
        assert (guard[:3 - shift] == 7).all() and (guard[3 - shift + n:] == 7).all()  # no stray writes


@pytest.mark.parametrize("spec", ["ddf:exact", "acwddf:minimax:window=5", "bvdf:rgb:window=7"])
def test_host_frame_stream(cuda, spec):
    """dfg_filter_host_frames: frames round-robin over three device slots
    (copies of frame f overlap the kernels of its neighbours); every frame
    must equal the oracle, for pinned and pageable buffers and frame counts
    below, at and above the slot count."""
    torch = cuda
    from paper_1009_0958_b200 import filter_host_frames
    s = parse_filter_spec(spec)
    for n, pinned in ((1, True), (3, False), (7, True)):
        imgs = [synth.noisy_image(75, 64, 30 + i, ("correlated", 0.2)) for i in range(n)]
        if pinned:
            ins = [torch.from_numpy(a).pin_memory().numpy() for a in imgs]
            outs = [torch.empty(a.shape, dtype=torch.uint8).pin_memory().numpy() for a in imgs]
        else:
            ins, outs = imgs, None
        got = filter_host_frames(ins, s, out=outs)
        for a, g in zip(imgs, got):
            assert (g == oracle.filter_image(a, s)).all(), (spec, n, pinned)
    assert filter_host_frames([], s) == []


@pytest.mark.parametrize("config", ["c1", "c2", "c3", "c4_bvdf_minimax", "c4_bvdf_rgb", "c4_ddf_minimax",
                                    "c4_ddf_rgb", "c5a", "c5b"])
def test_config_whole_frame_against_oracle(cuda, config):
    """Parity at the BASELINE full sizes, every pixel (SURVEY 8(d)
    "Correctness reporting"; the reference's own whole-image oracles,
    T/test_acceptance.py:169-195, T/test_filters.py:347-359): the config
    frame (C5b: all 64 frames) is filtered on the GPU exactly as bench.py
    does, the float64 oracle re-filters the whole frame on all host cores,
    and every mismatch must be a documented near-tie (relative gap < 1e-5),
    under 0.01 % of the pixels.  (So far every config has had 0.)"""
    torch = cuda
    cfg = synth.CONFIGS[config]
    s = parse_filter_spec(cfg["spec"])
    x = synth.config_input(config)
    if x.ndim == 4:
        got = filter_batch_device(torch.from_numpy(x).cuda(), s).cpu().numpy()
    else:
        got = filter_device(torch.from_numpy(x).cuda(), s).cpu().numpy()
    rep = oracle.parity_report(got, x, s)
    assert rep["checked_px"] == int(np.prod(x.shape[:-1])), rep
    assert rep["non_tie_mismatches"] == 0, (config, rep)
    assert rep["near_ties"] <= 1e-4 * rep["checked_px"], (config, rep)
    print(config, rep)


@pytest.mark.parametrize("spec", ["ddf:exact", "acwddf:minimax:window=5", "bvdf:rgb:window=7"])
@pytest.mark.parametrize("shape", [(6, 24001), (9000, 5), (2, 3), (1, 4097), (4097, 1)])
def test_extreme_aspect_ratios(cuda, spec, shape):
    """Very wide / very tall / tiny frames (grids with a single strip or a
    single tile row, windows larger than the image, both borders) through
    the device and host paths."""
    torch = cuda
    s = parse_filter_spec(spec)
    img = synth.noisy_image(*shape, 41, ("correlated", 0.2))
    for border in ("replicate", "reflect"):
        want = oracle.filter_image(img, s, border)
        got = filter_device(torch.from_numpy(img).cuda(), s, _policy(border)).cpu().numpy()
        assert (got == want).all(), (spec, shape, border, int((got != want).any(-1).sum()))
        assert (filter_host(img, s, _policy(border)) == want).all(), (spec, shape, border)


def test_apply_filter_float64_boundary(cuda):
    """The drop-in path (dfg_filter_host_f64): float64 RasterImage in, a new
    float64 RasterImage out, equal to the device path on a frame large
    enough for several host threads and row bands; values that are not
    integers in 0..255 raise ValueError (the GPU path's one input
    restriction) and leave no partial result."""
    torch = cuda
    img = synth.noisy_image(1030, 770, 7, ("correlated", 0.2))
    for spec in ("ddf:exact", "acwddf:minimax:window=5", "bvdf:rgb:window=7"):
        s = parse_filter_spec(spec)
        ri = RasterImage(img.astype(np.float64))
        out = apply_filter(ri, s)
        assert out.pixels.dtype == np.float64 and not np.shares_memory(out.pixels, ri.pixels)
        want = filter_device(torch.from_numpy(img).cuda(), s).cpu().numpy()
        assert (out.pixels == want).all(), spec
        assert apply_filter(ri, s, workers=4) == out
    base = img[:40, :50].astype(np.float64)
    for bad in (0.5, 256.0, -1.0, np.nan, np.inf, 255.0000001):
        a = base.copy()
        a[17, 23, 1] = bad
        with pytest.raises(ValueError):
            apply_filter(_raw_image(a), parse_filter_spec("ddf:exact"))
    with pytest.raises(ValueError):  # through a real RasterImage (it accepts non-integral values)
        apply_filter(RasterImage(base + 0.25), parse_filter_spec("ddf:exact"))


@pytest.mark.parametrize("spec,border", [("ddf:exact", "replicate"), ("acwddf:exact:window=5", "reflect"),
                                         ("ddf:exact:window=7", "replicate"), ("bvdf:minimax:window=9", "reflect")])
def test_float64_pipeline_bands(cuda, spec, border):
    """Large frames pipeline the float64 <-> uint8 conversions band by band
    around the device work (dfg_filter_host_f64 -> f64_pipeline): same
    pixels as the device path for 2 .. 16 bands (forced on a small frame
    through DFG_OPT_HOST_BANDS) and at the natural size; a bad value in the
    LAST band raises and leaves the caller's output untouched."""
    torch = cuda
    s = parse_filter_spec(spec)
    pol = _policy(border)
    H, W = (300, 211) if "window=9" not in spec else (140, 97)
    img = synth.noisy_image(H, W, 21, ("uncorrelated", 0.15))
    want = filter_device(torch.from_numpy(img).cuda(), s, pol).cpu().numpy()
    ri = RasterImage(img.astype(np.float64))
    for nb in (2, 3, 7, 16):
        with _lib.option("host_bands", nb):
            out = apply_filter(ri, s, pol)
        assert (out.pixels == want).all(), (spec, nb)
    a = img.astype(np.float64)
    a[H - 2, 5, 0] = 17.5
    with _lib.option("host_bands", 5), pytest.raises(ValueError):
        apply_filter(_raw_image(a), s, pol)
    with _lib.option("host_bands", 5):  # and the path is usable again afterwards
        assert (apply_filter(ri, s, pol).pixels == want).all()


def test_float64_pipeline_natural_size(cuda):
    torch = cuda
    s = parse_filter_spec("ddf:exact")
    img = synth.noisy_image(1500, 2100, 22, ("correlated", 0.2))  # 3 bands
    want = filter_device(torch.from_numpy(img).cuda(), s).cpu().numpy()
    out = apply_filter(RasterImage(img.astype(np.float64)), s)
    assert (out.pixels == want).all()


def _raw_image(a):
    """A duck-typed image carrying pixels RasterImage itself would reject
    (NaN / inf), to reach the C ABI's own validation."""
    class _Img:
        pixels = a
    return _Img()


@pytest.mark.parametrize("tma", [0, 1, 2, 3])
@pytest.mark.parametrize("spec", ["ddf:exact:window=7", "acwddf:minimax:window=5", "bvdf:rgb:window=5", "vmf:window=7"])
def test_tile_bulk_copies_on_and_off(cuda, spec, tma):
    """The CTA kernel's bulk tensor copies (DFG_OPT_TMA bit 0: each
    interior tile's region by TMA, prefetched a tile ahead; bit 1: the
    tile's colours out by a TMA store) give the same pixels as indexed
    loads / byte stores: 16-byte aligned rows (where the tensor maps apply),
    a 3-frame batch (3-D maps) and a strip at an interior row offset."""
    torch = cuda
    s = parse_filter_spec(spec)
    img = synth.noisy_image(160, 512, 13, ("correlated", 0.2))
    frames = np.stack([synth.noisy_image(70, 256, 50 + i, ("uncorrelated", 0.15)) for i in range(3)])
    with _lib.option("tma", tma):
        got = filter_device(torch.from_numpy(img).cuda(), s).cpu().numpy()
        gotb = filter_batch_device(torch.from_numpy(frames).cuda(), s).cpu().numpy()
        x = torch.from_numpy(img).cuda()
        gots = filter_rows_device(x[16:150], 160, 16, 40, 96, s).cpu().numpy()
    want = oracle.filter_image(img, s)
    assert (got == want).all(), (spec, tma, int((got != want).any(-1).sum()))
    for i in range(3):
        assert (gotb[i] == oracle.filter_image(frames[i], s)).all(), (spec, tma, i)
    assert (gots == want[40:136]).all(), (spec, tma)


def test_strip_job_cuda_kernel_single_rank_nccl(cuda):
    """parallel.filter_strips -- the step bench.py times at N > 1 -- with its
    default CUDA strip filter (dfg_filter_rows per row chunk) under a real
    NCCL group of one rank, gather on and off: equals the whole-frame call.
    (Several ranks need several GPUs; the collective logic itself is covered
    at world sizes 2..8 with gloo in tests/test_parallel.py, and a 4-rank
    partition is emulated here rank by rank through the same StripJob row
    bounds with hand-cut halos.)"""
    import socket

    import torch.distributed as dist

    from paper_1009_0958_b200.parallel import filter_strips, strip_rows

    torch = cuda
    spec = parse_filter_spec("ddf:exact:window=7")
    img = synth.noisy_image(700, 301, 31, ("correlated", 0.2))
    x = torch.from_numpy(img).cuda()
    want = filter_device(x, spec)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        for gather in (True, False):
            got = filter_strips(x, 0, 700, 700, spec, REPLICATE, gather=gather, chunks=4)
            torch.cuda.synchronize()
            assert (got == want).all(), gather
    finally:
        dist.destroy_process_group()
    # a 4-rank partition, one "rank" at a time on this GPU
    for rank in range(4):
        r0, r1, i0, i1 = strip_rows(700, 4, rank, 7)
        out = filter_rows_device(x[i0:i1].contiguous(), 700, i0, r0, r1 - r0, spec)
        assert (out == want[r0:r1]).all(), rank


@pytest.mark.parametrize("threads", [1, 3, 64])
def test_float64_path_thread_counts(cuda, threads):
    """dfg_filter_host_f64 with explicit host thread counts (the Python shim
    passes 0 = all cores), banded and unbanded: same pixels."""
    import ctypes

    torch = cuda
    spec = parse_filter_spec("acwddf:exact")
    img = synth.noisy_image(260, 190, 33, ("uncorrelated", 0.1))
    want = filter_device(torch.from_numpy(img).cuda(), spec).cpu().numpy().astype(np.float64)
    a = img.astype(np.float64)
    prm = _lib.params_from_spec(spec, "replicate")
    for nb in (0, 4):
        out = np.full(a.shape, -1.0)
        with _lib.option("host_bands", nb):
            rc = _lib.lib().dfg_filter_host_f64(a.ctypes.data_as(ctypes.c_void_p), 260, 190,
                                                out.ctypes.data_as(ctypes.c_void_p), ctypes.byref(prm), threads, None)
        _lib.check(rc)
        assert (out == want).all(), (threads, nb)
