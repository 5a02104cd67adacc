"""GPU parity: the CUDA path (through the C ABI) vs the oracle / golden vectors.

Bit-exact for fp32 outputs (bit patterns), raw int64 accumulators and argmax.
"""

import hashlib
from pathlib import Path

import numpy as np
import pytest

from cases import oracle_conv, random_conv_case
from conftest import cuda_ok
from golden_io import bits_equal, load_golden
from oracle import axemu_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


def _torch():
    import torch

    return torch


def _lut(entries, mode):
    from paper_2002_09481_b200 import types as T

    return T.MultLut(T.Signedness(mode), np.asarray(entries).astype(T.Signedness(mode).entry_dtype))


def gpu_conv(case, acc=True, force_generic=False, sm_limit=0, variant=0, ft_variant=0, use_ftable=True):
    """Run one case through ConvLayer (C-ABI stages: coeffs, quantize, [im2col], conv)."""
    torch = _torch()
    from paper_2002_09481_b200 import _lib
    from paper_2002_09481_b200.layer import ConvLayer
    from paper_2002_09481_b200.types import ConvGeometry, output_shape

    geo = ConvGeometry(case["strides"], case["dilations"], case["padding"])
    layer = ConvLayer(case["f"], case["f_range"], _lut(case["lut"], case["mode"]), geo,
                      round_mode=case["round_mode"], accumulator=case["accumulator"])
    layer.set_input_params(*case["in_range"])
    x = torch.from_numpy(case["x"]).cuda()
    flags = torch.zeros(2, dtype=torch.int32, device="cuda")
    acc_t = None
    if acc:
        acc_t = torch.empty(output_shape(case["x"].shape, case["f"].shape, geo), dtype=torch.int64, device="cuda")
    y = layer.run(x, None, out_flag=flags[0].data_ptr(), quant_flag=flags[1].data_ptr(),
                  force_generic=force_generic, sm_limit=sm_limit, variant=variant, acc_out=acc_t,
                  ft_variant=ft_variant, use_ftable=use_ftable)
    torch.cuda.synchronize()
    kernel = _lib.last_kernel()
    return y.cpu().numpy(), (acc_t.cpu().numpy() if acc else None), kernel


@pytest.mark.parametrize("path", ["ftable", "lut", "generic"])
def test_c1_cases_bit_exact(path):
    """The reference's 100 acceptance cases (seed 2026) through each conv kernel family:
    ftable (filter-specialised product table), lut (b-major LUT), generic (int64)."""
    g = load_golden("c1")
    rng = np.random.default_rng(2026)
    kernels = set()
    for i in range(100):
        case = random_conv_case(rng)
        y, acc, kern = gpu_conv(case, force_generic=path == "generic", use_ftable=path == "ftable")
        kernels.add(kern.split("<")[0])
        assert bits_equal(y, g[f"out_{i}"]), (i, kern)
        assert np.array_equal(acc, g[f"acc_{i}"]), (i, kern)
    if path == "generic":
        assert kernels == {"lutconv_generic"}
    elif path == "ftable":
        assert any(k.startswith("ft") for k in kernels), kernels
    else:
        assert not any(k.startswith("ft") for k in kernels) and "lutconv_generic" not in kernels, kernels


def test_all_ftable_variants_bit_identical():
    """Every ftable-kernel tile variant (pair-major and code-major tables) gives the oracle's bits
    (outputs and raw sums), including ragged pixel tiles, cout not a multiple of 16, residual +
    ReLU-free paths and both signedness."""
    from paper_2002_09481_b200 import _lib

    lib = _lib.load()
    nvar = lib.axb_ft_variant_count()
    rng = np.random.default_rng(78)
    cases = [random_conv_case(rng) for _ in range(16)]
    for mode in (O.SIGNED, O.UNSIGNED):
        big = dict(x=np.maximum(rng.standard_normal((5, 23, 21, 32)), 0).astype(np.float32),
                   f=rng.standard_normal((3, 3, 32, 61)).astype(np.float32), lut=O.random_lut(rng, mode),
                   mode=mode, padding="same", strides=(1, 1), dilations=(1, 1), accumulator=O.WRAP32,
                   round_mode=O.HALF_EVEN)
        big.update(in_range=(float(big["x"].min()), float(big["x"].max())),
                   f_range=(float(big["f"].min()), float(big["f"].max())))
        cases.append(big)
    cm_runs = 0
    for case in cases:
        want, want_acc = oracle_conv(case, return_acc=True)
        coutp = -(-case["f"].shape[3] // 16) * 16
        for v in range(1, nvar):
            lay = lib.axb_ft_variant_layout(v)
            if coutp % LAYOUT_BLOCK.get(lay, 16):  # code-major layouts: 32 / 64 / 32 / 16-channel blocks
                continue
            cm_runs += lay > 0
            y, acc, kern = gpu_conv(case, ft_variant=v)
            assert bits_equal(y, want), (v, kern)
            assert np.array_equal(acc, want_acc), (v, kern)
    assert cm_runs >= 12


def test_all_tile_variants_bit_identical():
    """Every fast-kernel tile variant (warps x pixels x channels) gives the same bits on seeded cases."""
    from paper_2002_09481_b200 import _lib

    nvar = _lib.load().axb_conv_variant_count()
    rng = np.random.default_rng(77)
    cases = [random_conv_case(rng) for _ in range(12)]
    big = dict(x=np.maximum(rng.standard_normal((3, 17, 19, 48)), 0).astype(np.float32),
               f=rng.standard_normal((3, 3, 48, 70)).astype(np.float32), lut=O.random_lut(rng, O.SIGNED),
               mode=O.SIGNED, padding="same", strides=(1, 1), dilations=(1, 1), accumulator=O.EXACT64,
               round_mode=O.HALF_EVEN)
    big.update(in_range=(float(big["x"].min()), float(big["x"].max())),
               f_range=(float(big["f"].min()), float(big["f"].max())))
    for case in cases + [big]:
        want, want_acc = oracle_conv(case, return_acc=True)
        for v in range(1, nvar):
            y, acc, kern = gpu_conv(case, variant=v)
            assert bits_equal(y, want), (v, kern)
            assert np.array_equal(acc, want_acc), (v, kern)


def test_c1_through_operator_api():
    """The reference-signature adapter (axconv2d) on the same 100 cases."""
    from paper_2002_09481_b200 import axconv2d
    from paper_2002_09481_b200 import types as T

    g = load_golden("c1")
    rng = np.random.default_rng(2026)
    for i in range(100):
        c = random_conv_case(rng)
        cfg = T.ConvConfig(geometry=T.ConvGeometry(c["strides"], c["dilations"], c["padding"]), chunk_size=c["chunk"],
                           accumulator=T.Accumulator(c["accumulator"]), round_mode=T.RoundMode(c["round_mode"]),
                           workers=c["workers"])
        y = axconv2d(T.Tensor4(c["x"]), T.Tensor4(c["f"], T.Layout.HWCN), T.Range(*c["in_range"]),
                     T.Range(*c["f_range"]), _lut(c["lut"], c["mode"]), cfg)
        assert bits_equal(y.data, g[f"out_{i}"]), i


def test_more_random_cases_vs_oracle():
    """Another 150 seeded cases (both kernels) against the pinned oracle."""
    rng = np.random.default_rng(31337)
    for i in range(150):
        case = random_conv_case(rng)
        want, want_acc = oracle_conv(case, return_acc=True)
        for generic in (False, True):
            y, acc, kern = gpu_conv(case, force_generic=generic)
            assert bits_equal(y, want), (i, kern)
            assert np.array_equal(acc, want_acc), (i, kern)


def test_extreme_ranges_kats():
    g = load_golden("kat")
    extremes = [((-1e6, 1e6), (-1e3, 1e3), O.SIGNED), ((0.0, 1e-9), (-1e-12, 1e-12), O.SIGNED),
                ((-1e-3, 1e5), (-7.0, 0.0), O.UNSIGNED), ((-9.0, -1.0), (-5.0, -0.1), O.UNSIGNED),
                ((0.0, 0.0), (3.0, 3.0), O.SIGNED)]
    for e, (ir, fr, mode) in enumerate(extremes):
        for rm in (O.HALF_AWAY, O.HALF_EVEN, O.TOWARD_ZERO):
            for acc in (O.EXACT64, O.WRAP32, O.SATURATE32):
                case = dict(x=g[f"ext{e}_x"], f=g[f"ext{e}_f"], in_range=ir, f_range=fr, lut=O.exact_lut(mode),
                            mode=mode, padding="same", strides=(1, 1), dilations=(1, 1), accumulator=acc,
                            round_mode=rm)
                for generic in (False, True):
                    y, _, _ = gpu_conv(case, acc=False, force_generic=generic)
                    assert bits_equal(y, g[f"ext{e}_{rm}_{acc}"]), (e, rm, acc, generic)


def test_overflow_kat_k33759():
    g = load_golden("kat")
    for acc in (O.EXACT64, O.WRAP32, O.SATURATE32):
        case = dict(x=np.ones((1, 33, 33, 31), np.float32), f=np.ones((33, 33, 31, 1), np.float32),
                    in_range=(0.0, 1.0), f_range=(0.0, 1.0), lut=np.full(65536, 65535, np.uint16),
                    mode=O.UNSIGNED, padding="valid", strides=(1, 1), dilations=(1, 1), accumulator=acc,
                    round_mode=O.HALF_AWAY)
        y, _, kern = gpu_conv(case, acc=False)
        assert bits_equal(y, g[f"ovf_{acc}"]), acc


def test_small_kats_and_config1():
    g = load_golden("kat")
    case = dict(x=np.zeros((1, 2, 2, 1), np.float32),
                f=np.array([0.4, -0.2, 0.7, -0.9], np.float32).reshape(2, 2, 1, 1), in_range=(0.0, 0.0),
                f_range=(-0.9, 0.7), lut=g["zero_in_entries"], mode=O.SIGNED, padding="valid", strides=(1, 1),
                dilations=(1, 1), accumulator=O.EXACT64, round_mode=O.HALF_AWAY)
    assert bits_equal(gpu_conv(case, acc=False)[0], g["zero_in_out"])
    case.update(x=g["asym_x"], f=g["asym_f"], in_range=(0.0, 1.0), f_range=(-2.0, 2.0),
                lut=O.exact_lut(O.UNSIGNED), mode=O.UNSIGNED, padding="same")
    assert bits_equal(gpu_conv(case, acc=False)[0], g["asym_out"])
    x1, f1 = g["cfg1_x"], g["cfg1_f"]
    for tag, lut in (("exact", O.exact_lut(O.SIGNED)), ("random", g["cfg1_rlut"])):
        case = dict(x=x1, f=f1, in_range=(float(x1.min()), float(x1.max())), f_range=(float(f1.min()), float(f1.max())),
                    lut=lut, mode=O.SIGNED, padding="same", strides=(1, 1), dilations=(1, 1), accumulator=O.EXACT64,
                    round_mode=O.HALF_AWAY)
        assert bits_equal(gpu_conv(case, acc=False)[0], g[f"cfg1_{tag}"])


def test_at_scale_first_layer_sha_and_grid_invariance():
    """1000x32x32x3 -> 16 (test_axconv.py:225-237): full output sha == reference; SM-count invariant."""
    g = load_golden("kat")
    rng = np.random.default_rng(8)
    xs = rng.uniform(0, 1, (1000, 32, 32, 3)).astype(np.float32)
    fs = rng.normal(0, 0.4, (3, 3, 3, 16)).astype(np.float32)
    case = dict(x=xs, f=fs, in_range=(0.0, 1.0), f_range=(-2.0, 2.0), lut=O.exact_lut(O.SIGNED), mode=O.SIGNED,
                padding="same", strides=(1, 1), dilations=(1, 1), accumulator=O.EXACT64, round_mode=O.HALF_AWAY)
    y, _, _ = gpu_conv(case, acc=False)
    assert hashlib.sha256(y.tobytes()).digest() == g["scale_sha"].tobytes()
    for lim in (1, 7, 64):
        y2, _, _ = gpu_conv(case, acc=False, sm_limit=lim)
        assert bits_equal(y, y2), lim


def test_quantize_kernel_codes_match_reference():
    """K2 alone: codes and zp padding vs the reference's quantize_values fixtures."""
    torch = _torch()
    from paper_2002_09481_b200 import _lib

    lib = _lib.load()
    g = load_golden("kat")
    rounds = [O.HALF_AWAY, O.HALF_EVEN, O.TOWARD_ZERO]
    s = torch.cuda.current_stream().cuda_stream
    for i in range(int(g["q_count"])):
        mn, mx = g[f"q{i}_range"]
        sgn, rm = (int(v) for v in g[f"q{i}_mode"])
        vals = g[f"q{i}_vals"]
        hp_ = _lib.QParams()
        _lib.check(lib.axb_coeffs_host(float(mn), float(mx), sgn, rm, hp_))
        assert (hp_.scale, hp_.zero_point) == (g[f"q{i}_coeffs"][0], int(g[f"q{i}_coeffs"][1]))
        prm = torch.zeros(_lib.QPARAMS_BYTES, dtype=torch.uint8, device="cuda")
        _lib.check(lib.axb_params_upload(hp_, prm.data_ptr(), s))
        x = torch.from_numpy(vals.reshape(1, 1, -1, 1)).cuda()
        n = vals.size
        codes = torch.empty((n + 2) * 16, dtype=torch.uint8, device="cuda")  # cs = 16, 1 pad col each side
        pixsum = torch.empty(n + 2, dtype=torch.int32, device="cuda")
        fl = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.check(lib.axb_quantize_pad(x.data_ptr(), 1, 1, n, 1, 0, 0, 1, 1, 16, prm.data_ptr(), sgn, rm,
                                        codes.data_ptr(), pixsum.data_ptr(), fl.data_ptr(), s))
        cb = codes.cpu().numpy().reshape(n + 2, 16)
        want = g[f"q{i}_codes"]
        assert np.array_equal(cb[1:-1, 0].view(np.int8 if sgn else np.uint8), want), i
        assert (cb[[0, -1], 0] == (hp_.zero_point & 0xFF)).all()
        assert (cb[:, 1:] == 0).all()
        assert np.array_equal(pixsum.cpu().numpy()[1:-1], want.astype(np.int32))


def test_range_kernel_exact_and_nonfinite():
    torch = _torch()
    from paper_2002_09481_b200 import _lib

    lib = _lib.load()
    s = torch.cuda.current_stream().cuda_stream
    rng = np.random.default_rng(4)
    for n in (1, 3, 17, 1000, 1 << 20, (1 << 22) + 5):
        x = (rng.standard_normal(n) * 10).astype(np.float32)
        for off in ((0,) if n == 1 else (0, 1)):
            xt = torch.from_numpy(x).cuda()[off:]
            r = torch.empty(2, dtype=torch.int32, device="cuda")
            fl = torch.zeros(1, dtype=torch.int32, device="cuda")
            _lib.check(lib.axb_range_reset(r.data_ptr(), s))
            _lib.check(lib.axb_range_minmax(xt.data_ptr(), xt.numel(), r.data_ptr(), fl.data_ptr(), s))
            mn, mx, f = _lib.c_vp(), None, None
            a, b, c = (np.zeros(1, np.float32), np.zeros(1, np.float32), np.zeros(1, np.int32))
            _lib.check(lib.axb_range_read(r.data_ptr(), fl.data_ptr(), a.ctypes.data, b.ctypes.data, c.ctypes.data, s))
            assert a[0] == x[off:].min() and b[0] == x[off:].max() and c[0] == 0
    x = np.ones(1000, np.float32)
    x[517] = np.inf
    xt = torch.from_numpy(x).cuda()
    r = torch.empty(2, dtype=torch.int32, device="cuda")
    fl = torch.zeros(1, dtype=torch.int32, device="cuda")
    lib.axb_range_reset(r.data_ptr(), s)
    lib.axb_range_minmax(xt.data_ptr(), 1000, r.data_ptr(), fl.data_ptr(), s)
    assert int(fl.item()) & _lib.FLAG_NONFINITE


def test_operator_errors_match_reference():
    from paper_2002_09481_b200 import axconv2d
    from paper_2002_09481_b200 import types as T

    lut = T.exact_lut(T.Signedness.UNSIGNED)
    x = T.Tensor4(np.zeros((1, 4, 4, 2), np.float32))
    f = T.Tensor4(np.zeros((3, 3, 3, 1), np.float32), T.Layout.HWCN)
    with pytest.raises(ValueError, match="channels"):
        axconv2d(x, f, T.Range(0, 1), T.Range(0, 1), lut, T.ConvConfig())
    xn = np.ones((1, 4, 4, 1), np.float32)
    xn[0, 1, 1, 0] = np.nan
    with pytest.raises(ValueError, match="finite"):
        axconv2d(T.Tensor4(xn), T.Tensor4(np.ones((2, 2, 1, 1), np.float32), T.Layout.HWCN), T.Range(0, 1),
                 T.Range(0, 1), lut, T.ConvConfig())
    out = axconv2d(T.Tensor4(np.zeros((0, 4, 4, 1), np.float32)), T.Tensor4(np.ones((2, 2, 1, 3), np.float32),
                   T.Layout.HWCN), T.Range(0, 1), T.Range(0, 1), lut, T.ConvConfig())
    assert out.shape == (0, 3, 3, 3)
    with pytest.raises(ValueError, match="HWCN"):
        axconv2d(x, T.Tensor4(np.zeros((3, 3, 2, 1), np.float32)), T.Range(0, 1), T.Range(0, 1), lut, T.ConvConfig())


NETS = [("r8_trunc2", "r8", 1, 0, ("t", 2)), ("r8_random", "r8", 1, 0, ("r",)),
        ("r8_unsigned", "r8", 1, 3, ("tu", 1)), ("r62_trunc3", "r62", 10, 1, ("t", 3)),
        ("r50_exact", "r50", 0, 0, ("e",))]


@pytest.mark.parametrize("tag,arch,depth,seed,kind", NETS)
def test_graph_end_to_end_bit_exact(tag, arch, depth, seed, kind):
    """GPU executor (fused epilogues, device ranges) vs reference graph.run: logits, argmax, every conv."""
    torch = _torch()
    from paper_2002_09481_b200 import resnet
    from paper_2002_09481_b200 import types as T
    from paper_2002_09481_b200.graph import GpuGraph

    g = load_golden("nets")
    if kind[0] == "t":
        lut = T.truncated_lut(T.Signedness.SIGNED, kind[1])
    elif kind[0] == "tu":
        lut = T.truncated_lut(T.Signedness.UNSIGNED, kind[1])
    elif kind[0] == "e":
        lut = T.exact_lut(T.Signedness.SIGNED)
    else:
        lut = T.MultLut(T.Signedness.SIGNED, g["random_lut_seed123"])
    nodes = resnet.resnet50(lut, seed=seed) if arch == "r50" else resnet.cifar_resnet(depth, lut, seed=seed)
    gg = GpuGraph(nodes)
    trace = {}
    y = gg.run(torch.from_numpy(g[f"{tag}_x"]).cuda(), trace=trace).cpu().numpy()
    ids = list(g[f"{tag}_conv_ids"])
    for cid, want in zip(ids, g[f"{tag}_conv_sha"]):
        # the fused epilogue may have absorbed Add/ReLU; compare the conv node's own value only when unfused
        plan = gg.conv_plans[cid]
        if plan.relu or plan.residual is not None:  # value is post-Add/ReLU (fused); logits cover it
            continue
        got = hashlib.sha256(np.ascontiguousarray(trace[cid].cpu().numpy()).tobytes()).digest()
        assert got == want.tobytes(), cid
    assert bits_equal(y, g[f"{tag}_logits"])
    assert np.array_equal(y.reshape(y.shape[0], -1).argmax(1), g[f"{tag}_argmax"])


def _bench_config(arch):
    from paper_2002_09481_b200 import datasets, resnet
    from paper_2002_09481_b200 import types as T

    lut = T.truncated_lut(T.Signedness.SIGNED, 2)
    if arch == "r8":  # BASELINE config 2, bench.py --workload r8, rank 0's batch
        return resnet.cifar_resnet(1, lut, seed=0), datasets.synthetic_cifar10(1024, seed=1000)[0]
    if arch == "mbv1":  # config 5's depthwise conv in a MobileNet-v1-shaped net, bench.py --workload mbv1
        return resnet.mobilenet_v1(lut, seed=0), datasets.synthetic_imagenet(256, seed=1000)[0]
    return resnet.resnet50(lut, seed=0), datasets.synthetic_imagenet(256, seed=1000)[0]  # config 3 (default)


def _sha(t) -> bytes:
    return hashlib.sha256(np.ascontiguousarray(t.cpu().numpy()).tobytes()).digest()


@pytest.mark.parametrize("arch", ["r8", "r50", "mbv1"])
def test_benchmarked_configs_bit_exact_vs_reference(arch):
    """The benchmarked networks at their full batch -- ResNet-8 b1024, ResNet-50 224x224 b256 and the
    MobileNet-v1-shaped net b256 (13 depthwise layers: per-channel reference axconv2d) with
    truncated_lut(signed, 2), calibrated weights -- against the REAL reference graph.run on the same
    batch (tests/golden/bench.npz): every unfused conv output, all logits, argmax.  Then again after the
    per-layer autotune, through the captured CUDA graph (bench.py's timed path)."""
    torch = _torch()
    from paper_2002_09481_b200.graph import GpuGraph

    g = load_golden("bench")
    nodes, x = _bench_config(arch)
    gg = GpuGraph(nodes)
    xd = torch.from_numpy(x).cuda()
    trace = {}
    y = gg.run(xd, trace=trace)
    checked = 0
    for cid, want in zip(g[f"{arch}_conv_ids"], g[f"{arch}_conv_sha"]):
        plan = gg.conv_plans[str(cid)]
        if plan.relu or plan.residual is not None:  # fused Add/ReLU: covered by the logits
            continue
        assert _sha(trace[str(cid)]) == want.tobytes(), cid
        checked += 1
    assert checked >= 1
    del trace
    assert _sha(y) == g[f"{arch}_logits_sha"].tobytes()
    am = y.reshape(y.shape[0], -1).argmax(1).cpu().numpy()
    assert np.array_equal(am, g[f"{arch}_argmax"])
    gg.autotune(xd)
    gg.capture(tuple(xd.shape))
    y2 = gg.replay(xd)
    assert _sha(y2) == g[f"{arch}_logits_sha"].tobytes()


def test_sweep_first_candidate_full_batch_vs_reference():
    """Config 4 at bench.py's sweep batch: ResNet-62 with the first candidate table (truncated_lut(signed,
    0)) on synthetic_cifar10(1000, 1000) -- all 1000 logits rows bit-identical to the real reference's
    graph.run (tests/golden/bench.npz r62sweep_logits_sha).  (This deep random network's argmax is one
    class for every image; the check is the logits' bits.)"""
    import sys

    torch = _torch()
    from paper_2002_09481_b200 import datasets, resnet
    from paper_2002_09481_b200.graph import GpuGraph

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import bench

    g = load_golden("bench")
    x = datasets.synthetic_cifar10(1000, seed=1000)[0]
    y = GpuGraph(resnet.cifar_resnet(10, bench.sweep_luts()[0], seed=0)).run(torch.from_numpy(x).cuda())
    assert _sha(y) == g["r62sweep_logits_sha"].tobytes()
    assert np.array_equal(y.reshape(1000, -1).argmax(1).cpu().numpy(), g["r62sweep_argmax"])


def test_r50_exact_lut_full_batch_vs_reference():
    """Config 5 control at the ResNet-50 shape: the benchmarked ResNet-50 b256 with exact_lut(signed)
    (bench.py --lut exact) -- all 256 logits rows and the argmax bit-identical to the real reference's
    graph.run on the same batch and weights (tests/golden/bench.npz r50exact_*)."""
    torch = _torch()
    from paper_2002_09481_b200 import datasets, resnet
    from paper_2002_09481_b200 import types as T
    from paper_2002_09481_b200.graph import GpuGraph

    g = load_golden("bench")
    assert "r50exact_logits_sha" in g
    x = datasets.synthetic_imagenet(256, seed=1000)[0]
    y = GpuGraph(resnet.resnet50(T.exact_lut(T.Signedness.SIGNED), seed=0)).run(torch.from_numpy(x).cuda())
    assert _sha(y) == g["r50exact_logits_sha"].tobytes()
    assert np.array_equal(y.reshape(256, -1).argmax(1).cpu().numpy(), g["r50exact_argmax"])


def test_r50_full_batch_grid_invariant():
    """ResNet-50 at 256 images on a 100-SM persistent grid (other tile-to-CTA assignment) gives the
    reference's bits (the grid size must never change results)."""
    torch = _torch()
    from paper_2002_09481_b200.graph import GpuGraph

    g = load_golden("bench")
    nodes, x = _bench_config("r50")
    y = GpuGraph(nodes, sm_limit=100).run(torch.from_numpy(x).cuda())
    assert _sha(y) == g["r50_logits_sha"].tobytes()


def test_exact_lut_control_full_size_layer():
    """Config 5 control: exact-LUT accumulators == exact fp64 GEMM on the codes (|A| < 2^53), R50 3x3x64 layer."""
    torch = _torch()
    import torch.nn.functional as F

    rng = np.random.default_rng(9)
    x = np.maximum(rng.standard_normal((16, 56, 56, 64)), 0).astype(np.float32)
    f = (rng.standard_normal((3, 3, 64, 64)) * 0.06).astype(np.float32)
    for mode in (O.SIGNED, O.UNSIGNED):
        case = dict(x=x, f=f, in_range=(float(x.min()), float(x.max())), f_range=(float(f.min()), float(f.max())),
                    lut=O.exact_lut(mode), mode=mode, padding="same", strides=(1, 1), dilations=(1, 1),
                    accumulator=O.EXACT64, round_mode=O.HALF_AWAY)
        _, acc, kern = gpu_conv(case)
        assert kern != "lutconv_generic"
        s1, z1 = O.compute_coeffs(*case["in_range"], mode)
        s2, z2 = O.compute_coeffs(*case["f_range"], mode)
        xc = torch.from_numpy(O.quantize_values(x, s1, z1, mode).astype(np.float64)).cuda()
        fc = torch.from_numpy(O.quantize_values(f, s2, z2, mode).astype(np.float64)).cuda()
        xp = F.pad(xc.permute(0, 3, 1, 2), (1, 1, 1, 1), value=float(z1))
        want = F.conv2d(xp, fc.permute(3, 2, 0, 1)).permute(0, 2, 3, 1)
        assert torch.equal(torch.from_numpy(acc).cuda().double(), want)


@pytest.mark.parametrize("stride,shape,mode", [(1, (4, 28, 28, 32), O.SIGNED), (2, (4, 28, 28, 48), O.UNSIGNED),
                                               (1, (2, 14, 14, 128), O.SIGNED), (1, (2, 112, 112, 32), O.SIGNED),
                                               (2, (2, 112, 112, 32), O.UNSIGNED), (1, (2, 56, 56, 128), O.UNSIGNED),
                                               (2, (2, 56, 56, 128), O.SIGNED), (1, (3, 7, 9, 40), O.SIGNED)])
def test_depthwise_matches_per_channel_oracle(stride, shape, mode):
    """Config 5: depthwise approximate conv == per-channel axconv2d with shared ranges (bit-exact), at the
    MobileNet shapes (n,112,112,32) and (n,56,56,128), stride 1 and 2, ragged channel blocks (40, 48):
    the channel-bank table kernels (row-strip depthwise_rs, per-pixel depthwise_ct) and the b-major LUT
    kernel, outputs and raw sums."""
    torch = _torch()
    from paper_2002_09481_b200.layer import ConvLayer
    from paper_2002_09481_b200.types import ConvGeometry

    rng = np.random.default_rng(stride * 100 + shape[3])
    x = np.maximum(rng.standard_normal(shape), 0).astype(np.float32)
    f = (rng.standard_normal((3, 3, shape[3], 1)) * 0.3).astype(np.float32)
    bias = (rng.standard_normal(shape[3]) * 0.05).astype(np.float32)
    lut = O.random_lut(rng, mode)
    ir, fr = (float(x.min()), float(x.max())), (float(f.min()), float(f.max()))
    want = np.concatenate([O.axconv2d(x[..., c:c + 1], f[:, :, c:c + 1, :], ir, fr, lut, mode, padding="same",
                                      strides=(stride, stride)) for c in range(shape[3])], axis=3)
    want = (want + bias).astype(np.float32)
    layer = ConvLayer(f, fr, _lut(lut, mode), ConvGeometry((stride, stride), (1, 1), "same"), bias=bias,
                      depthwise=True)
    layer.set_input_params(*ir)
    flags = torch.zeros(2, dtype=torch.int32, device="cuda")
    _, want_acc = O.depthwise_conv(x, f, ir, fr, lut, mode, padding="same", strides=(stride, stride),
                                   return_acc=True)
    from paper_2002_09481_b200 import _lib

    for use_table, variant, kern in ((True, 0, "depthwise_rs"), (True, 1, "depthwise_ct"),
                                     (False, 0, "depthwise_lut")):
        acc = torch.empty(want_acc.shape, dtype=torch.int64, device="cuda")
        y = layer.run(torch.from_numpy(x).cuda(), None, out_flag=flags[0].data_ptr(),
                      quant_flag=flags[1].data_ptr(), use_ftable=use_table, acc_out=acc, variant=variant)
        assert _lib.last_kernel() == kern
        assert bits_equal(y.cpu().numpy(), want), kern
        assert np.array_equal(acc.cpu().numpy(), want_acc), kern


def test_quantizer_fast_path_sweep():
    """quantize_pad (fp32 estimate + tie fallback) vs quantize_values on dense near-tie sweeps:
    values within a few ulps of every half-step and every integer step, random ranges, all modes,
    plus out-of-range values (clipping) -- bit-exact codes and pixel sums."""
    torch = _torch()
    from paper_2002_09481_b200 import _lib

    lib = _lib.load()
    s = torch.cuda.current_stream().cuda_stream
    rng = np.random.default_rng(77)
    rounds = {O.HALF_AWAY: 0, O.HALF_EVEN: 1, O.TOWARD_ZERO: 2}
    for trial in range(24):
        mode = (O.SIGNED, O.UNSIGNED)[trial % 2]
        rname = list(rounds)[trial % 3]
        mn = float(-abs(rng.standard_normal()) * 10 ** rng.uniform(-3, 3)) if trial % 4 else 0.0
        mx = float(abs(rng.standard_normal()) * 10 ** rng.uniform(-3, 3))
        scale, zp = O.compute_coeffs(mn, mx, mode, rname)
        lo, _ = O.bounds(mode)
        k = np.arange(-300, 300, dtype=np.float64)
        base = np.concatenate([(k + 0.5 - zp + lo) * scale, (k - zp + lo) * scale]).astype(np.float32)
        ulps = np.arange(-3, 4, dtype=np.int32)
        near = (base.view(np.int32)[:, None] + ulps[None, :]).reshape(-1).view(np.float32)
        vals = np.concatenate([near, rng.uniform(mn * 1.5, mx * 1.5, 50000).astype(np.float32)])
        vals = vals[np.isfinite(vals)]
        hp_ = _lib.QParams()
        _lib.check(lib.axb_coeffs_host(mn, mx, int(mode == O.SIGNED), rounds[rname], hp_))
        prm = torch.zeros(_lib.QPARAMS_BYTES, dtype=torch.uint8, device="cuda")
        _lib.check(lib.axb_params_upload(hp_, prm.data_ptr(), s))
        for c in (4, 16, 64):  # 4: per-word kernel; 16, 64: 16-channel-chunk kernel
            v = vals[: len(vals) // c * c]
            want = O.quantize_values(v, scale, zp, mode, rname)
            n = len(v) // c
            cs = max(16, c)
            x = torch.from_numpy(v.reshape(1, 1, n, c)).cuda()
            codes = torch.empty(n * cs, dtype=torch.uint8, device="cuda")
            pixsum = torch.empty(n, dtype=torch.int32, device="cuda")
            fl = torch.zeros(1, dtype=torch.int32, device="cuda")
            _lib.check(lib.axb_quantize_pad(x.data_ptr(), 1, 1, n, c, 0, 0, 0, 0, cs, prm.data_ptr(),
                                            int(mode == O.SIGNED), rounds[rname], codes.data_ptr(), pixsum.data_ptr(),
                                            fl.data_ptr(), s))
            cb = codes.cpu().numpy().reshape(n, cs)
            got = cb[:, :c].reshape(-1).view(np.int8 if mode == O.SIGNED else np.uint8)
            assert np.array_equal(got, want), (trial, c, mode, rname, np.flatnonzero(got != want)[:5])
            assert (cb[:, c:] == 0).all()
            assert np.array_equal(pixsum.cpu().numpy(), want.reshape(n, c).astype(np.int32).sum(1)), (trial, c)
            assert int(fl.item()) == 0
            # the fused path: coefficients of a device range computed in the kernel prologue
            mn32, mx32 = np.float32(mn), np.float32(mx)
            s2, zp2 = O.compute_coeffs(float(mn32), float(mx32), mode, rname)
            want2 = O.quantize_values(v, s2, zp2, mode, rname)
            ordv = np.array([mn32, mx32], np.float32).view(np.int32)
            ordv = np.where(ordv >= 0, ordv, ordv ^ 0x7FFFFFFF).astype(np.int32)
            rng_d = torch.from_numpy(ordv).cuda()
            prm2 = torch.zeros(_lib.QPARAMS_BYTES, dtype=torch.uint8, device="cuda")
            _lib.check(lib.axb_quantize_pad_range(x.data_ptr(), 1, 1, n, c, 0, 0, 0, 0, cs, rng_d.data_ptr(),
                                                  int(mode == O.SIGNED), rounds[rname], prm2.data_ptr(),
                                                  codes.data_ptr(), pixsum.data_ptr(), fl.data_ptr(), s))
            cb = codes.cpu().numpy().reshape(n, cs)
            got = cb[:, :c].reshape(-1).view(np.int8 if mode == O.SIGNED else np.uint8)
            assert np.array_equal(got, want2), (trial, c, "range", np.flatnonzero(got != want2)[:5])
            assert np.array_equal(pixsum.cpu().numpy(), want2.reshape(n, c).astype(np.int32).sum(1))
            pb = prm2.cpu().numpy()
            assert pb[:8].view(np.float64)[0] == s2 and pb[8:12].view(np.int32)[0] == zp2


def test_cifar_decode_kernel_matches_reference_decode():
    """axb_cifar_decode == the reference's load_cifar10 decode (formats.py:138-157) bit for bit,
    with the fused input range and the label check."""
    torch = _torch()
    from paper_2002_09481_b200 import _lib
    from paper_2002_09481_b200 import formats as F
    from paper_2002_09481_b200.datasets import synthetic_cifar10

    lib = _lib.load()
    g = load_golden("formats")
    imgs, labels = synthetic_cifar10(1000, seed=4)
    for rec, want_img, want_lab in ((g["cifar_records"].reshape(-1, 3073), g["cifar_images"], g["cifar_labels"]),
                                    (F.encode_cifar10(imgs, labels), imgs, labels)):
        n = rec.shape[0]
        d_rec = torch.from_numpy(np.ascontiguousarray(rec)).cuda()
        out = torch.empty((n, 32, 32, 3), dtype=torch.float32, device="cuda")
        lab = torch.empty(n, dtype=torch.uint8, device="cuda")
        rng = torch.tensor([2**31 - 1, -(2**31)], dtype=torch.int32, device="cuda")
        flags = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.check(lib.axb_cifar_decode(d_rec.data_ptr(), n, out.data_ptr(), lab.data_ptr(), rng.data_ptr(),
                                        flags.data_ptr(), None))
        torch.cuda.synchronize()
        assert bits_equal(out.cpu().numpy(), want_img)
        assert np.array_equal(lab.cpu().numpy(), want_lab)
        mn, mx = (float(np.float32(v)) for v in (want_img.min(), want_img.max()))
        r = rng.cpu().numpy()
        got = [np.int32(v) for v in r]
        ords = [int(v) if v >= 0 else int(v) ^ 0x7FFFFFFF for v in got]
        assert np.array(ords, np.int32).view(np.float32).tolist() == [mn, mx]
        assert int(flags.item()) == 0
    bad = np.zeros((3, 3073), np.uint8)
    bad[2, 0] = 12
    d_rec = torch.from_numpy(bad).cuda()
    out = torch.empty((3, 32, 32, 3), dtype=torch.float32, device="cuda")
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.check(lib.axb_cifar_decode(d_rec.data_ptr(), 3, out.data_ptr(), None, None, flags.data_ptr(), None))
    assert int(flags.item()) & _lib.FLAG_LABEL


def test_graph_on_cifar_records_matches_images():
    """GpuGraph fed CIFAR-10 records (device decode, fused range) gives the same logits bits as
    fed the decoded fp32 images -- eagerly, replayed, and through run_pipelined from host."""
    torch = _torch()
    from paper_2002_09481_b200 import formats as F
    from paper_2002_09481_b200 import resnet
    from paper_2002_09481_b200 import types as T
    from paper_2002_09481_b200.datasets import synthetic_cifar10
    from paper_2002_09481_b200.graph import GpuGraph

    imgs, labels = synthetic_cifar10(96, seed=21)
    rec = F.encode_cifar10(imgs, labels)
    g = GpuGraph(resnet.cifar_resnet(1, T.truncated_lut(T.Signedness.SIGNED, 2), seed=0))
    want = g.run(torch.from_numpy(imgs).cuda()).cpu().numpy()
    got = g.run(torch.from_numpy(rec).cuda()).cpu().numpy()
    assert bits_equal(got, want)
    assert np.array_equal(g.labels.cpu().numpy(), labels)
    hosts = [torch.from_numpy(rec).pin_memory() for _ in range(3)]
    outs = g.run_pipelined(hosts)
    for o in outs:
        assert bits_equal(o.numpy(), want)
    bad = rec.copy()
    bad[5, 0] = 11
    with pytest.raises(F.FormatError, match="label"):
        g.run(torch.from_numpy(bad).cuda())


@pytest.mark.parametrize("mode", [O.SIGNED, O.UNSIGNED])
def test_fused_quantize_im2col_equals_two_pass(mode):
    """axb_quantize_im2col (one pass, fp32 -> code rows) == axb_quantize_pad + axb_im2col_pack ==
    the oracle's im2cols (code rows + patch sums), with host parameters and with in-kernel
    coefficients of a device range."""
    torch = _torch()
    from paper_2002_09481_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(5)
    for (n, h, w, c, kh, kw, s, d, pads) in [(3, 17, 13, 3, 3, 3, 1, 1, (1, 1, 1, 1)), (2, 23, 23, 3, 7, 7, 2, 1, (3, 3, 3, 3)),
                                              (4, 9, 11, 5, 3, 2, 2, 2, (0, 2, 1, 0)), (1, 8, 8, 1, 5, 5, 1, 1, (2, 2, 2, 2)),
                                              (2, 40, 37, 13, 7, 7, 2, 2, (6, 6, 6, 6)),  # patch > smem: two-pass path
                                              (3, 70, 66, 3, 3, 3, 1, 1, (1, 1, 1, 1))]:  # several tiles per image
        x = rng.uniform(-1.5, 2.5, (n, h, w, c)).astype(np.float32)
        x[0, 0, 0, 0] = 0.5  # a few exact half-steps / ties
        pt, pb, pl, pr = pads
        hp, wp = h + pt + pb, w + pl + pr
        oh, ow = (hp - ((kh - 1) * d + 1)) // s + 1, (wp - ((kw - 1) * d + 1)) // s + 1
        cs = int(lib.axb_channel_stride(c))
        kp = int(lib.axb_conv_im2col_kp(c, kh, kw))
        xd = torch.from_numpy(x).cuda()
        rngd = torch.tensor([np.float32(x.min()).view(np.int32), np.float32(x.max()).view(np.int32)], dtype=torch.int32,
                            device="cuda")
        rngd = torch.where(rngd >= 0, rngd, rngd ^ 0x7FFFFFFF)
        sgn = int(mode == O.SIGNED)
        for use_range in (False, True):
            params = torch.zeros(2, _lib.QPARAMS_BYTES, dtype=torch.uint8, device="cuda")
            if not use_range:
                hpq = _lib.QParams()
                _lib.check(lib.axb_coeffs_host(float(x.min()), float(x.max()), sgn, 0, hpq))
                _lib.check(lib.axb_params_upload(hpq, params[0].data_ptr(), None))
                _lib.check(lib.axb_params_upload(hpq, params[1].data_ptr(), None))
            codes = torch.empty(n * hp * wp * cs, dtype=torch.uint8, device="cuda")
            pix = torch.empty(n * hp * wp, dtype=torch.int32, device="cuda")
            fl = torch.zeros(2, dtype=torch.int32, device="cuda")
            r_ptr = rngd.data_ptr() if use_range else None
            if use_range:
                _lib.check(lib.axb_quantize_pad_range(xd.data_ptr(), n, h, w, c, pt, pb, pl, pr, cs, r_ptr, sgn, 0,
                                                      params[0].data_ptr(), codes.data_ptr(), pix.data_ptr(),
                                                      fl.data_ptr(), None))
            else:
                _lib.check(lib.axb_quantize_pad(xd.data_ptr(), n, h, w, c, pt, pb, pl, pr, cs, params[0].data_ptr(),
                                                sgn, 0, codes.data_ptr(), pix.data_ptr(), fl.data_ptr(), None))
            rows1 = torch.empty(n * oh * ow * kp, dtype=torch.uint8, device="cuda")
            sum1 = torch.empty(n * oh * ow, dtype=torch.int32, device="cuda")
            _lib.check(lib.axb_im2col_pack(codes.data_ptr(), n, hp, wp, cs, c, kh, kw, s, s, d, d, oh, ow, kp, sgn,
                                           rows1.data_ptr(), sum1.data_ptr(), None))
            rows2 = torch.empty_like(rows1)
            sum2 = torch.empty_like(sum1)
            _lib.check(lib.axb_quantize_im2col(xd.data_ptr(), n, h, w, c, pt, pl, kh, kw, s, s, d, d, oh, ow, kp,
                                               r_ptr, params[1].data_ptr(), sgn, 0, rows2.data_ptr(),
                                               sum2.data_ptr(), fl[1:].data_ptr(), None))
            torch.cuda.synchronize()
            assert torch.equal(rows1, rows2), (n, h, w, c, kh, kw, use_range)
            assert torch.equal(sum1, sum2)
            assert int(fl[1].item()) == 0
            # and both equal the oracle's im2cols (axconv.py:160-196): code rows (raw bytes, zero beyond K)
            # and patch sums
            sc, zp = O.compute_coeffs(float(x.min()), float(x.max()), mode)
            mat, sums = O.im2cols(x, sc, zp, mode, O.HALF_AWAY, kh, kw, pads, (s, s), (d, d))
            kk = kh * kw * c
            got = rows2.cpu().numpy().reshape(-1, kp)
            assert np.array_equal(got[:, :kk], mat.view(np.uint8)) and not got[:, kk:].any()
            assert np.array_equal(sum2.cpu().numpy(), sums)


def test_graph_autotune_keeps_bits():
    """Per-layer kernel autotune (every ftable variant and the b-major LUT kernel timed on live
    activations, bits compared inside) leaves the logits bit-identical to the cost-model run; a
    forced LUT-kernel pick (tuning value -1) runs that kernel with the same bits."""
    torch = _torch()
    from paper_2002_09481_b200 import resnet
    from paper_2002_09481_b200 import types as T
    from paper_2002_09481_b200.datasets import synthetic_cifar10
    from paper_2002_09481_b200.graph import GpuGraph

    imgs, _ = synthetic_cifar10(64, seed=33)
    g = GpuGraph(resnet.cifar_resnet(1, T.truncated_lut(T.Signedness.SIGNED, 2), seed=0))
    x = torch.from_numpy(imgs).cuda()
    want = g.run(x).cpu().numpy()
    picks = g.autotune(x, reps=1)
    assert len(picks) == 10 and all(v.startswith(("ft", "cm", "c16", "c32", "c64")) or v == "lut_bmajor"
                                    for v in picks.values()), picks
    # only the table layout each layer's pick reads stays resident
    for p in g.conv_plans.values():
        assert p.layer.ftable is None or p.layer.ftable_cm is None, p.node["id"]
    assert bits_equal(g.run(x).cpu().numpy(), want)
    g.set_tuning({nid: -1 for nid in g.tuning()})
    prof = []
    assert bits_equal(g.run(x, profile=prof).cpu().numpy(), want)
    assert {fam for *_, fam in prof} == {"lutconv_fast"}, {fam for *_, fam in prof}


def test_operator_api_large_call_uses_ftable_bit_exact():
    """torch_axconv2d on the 1000-image first layer (test_axconv.py:225-237): large calls build the
    filter-specialised table per call; output sha == the reference's."""
    torch = _torch()
    from paper_2002_09481_b200 import _lib
    from paper_2002_09481_b200.axconv import torch_axconv2d
    from paper_2002_09481_b200.types import ConvGeometry

    g = load_golden("kat")
    rng = np.random.default_rng(8)
    xs = rng.uniform(0, 1, (1000, 32, 32, 3)).astype(np.float32)
    fs = rng.normal(0, 0.4, (3, 3, 3, 16)).astype(np.float32)
    y = torch_axconv2d(torch.from_numpy(xs).cuda(), torch.from_numpy(fs).cuda(), (0.0, 1.0), (-2.0, 2.0),
                       _lut(O.exact_lut(O.SIGNED), O.SIGNED), ConvGeometry(padding="same"))
    assert _lib.last_kernel().startswith("ft"), _lib.last_kernel()
    assert hashlib.sha256(y.cpu().numpy().tobytes()).digest() == g["scale_sha"].tobytes()


def test_reference_model_file_runs_bit_exact(tmp_path):
    """A model file written by the reference (transform + save_model) loads with model.load_model
    and runs on the GPU executor with the reference executor's logits, bit for bit."""
    torch = _torch()
    from paper_2002_09481_b200 import types as T
    from paper_2002_09481_b200.formats import save_lut
    from paper_2002_09481_b200.graph import GpuGraph
    from paper_2002_09481_b200.model import load_model

    g = load_golden("formats")
    (tmp_path / "ax.json").write_bytes(g["model_json"].tobytes())
    (tmp_path / "ax.weights.bin").write_bytes(g["model_weights"].tobytes())
    save_lut(T.truncated_lut(T.Signedness.SIGNED, 2), tmp_path / "ax.axm")
    nodes = load_model(tmp_path / "ax.json")
    y = GpuGraph(nodes).run(torch.from_numpy(g["model_input"]).cuda()).cpu().numpy()
    assert bits_equal(y, g["model_logits"])


def test_r50_autotune_all_variants_agree():
    """Regression for a write-after-read race between LDS reads of a ring stage and the TMA refill
    (fixed with fence.proxy.async before the release): autotune compares every ftable variant's
    bits on every ResNet-50 layer at batch 128, twice."""
    torch = _torch()
    from paper_2002_09481_b200 import datasets, resnet
    from paper_2002_09481_b200 import types as T
    from paper_2002_09481_b200.graph import GpuGraph

    g = GpuGraph(resnet.resnet50(T.truncated_lut(T.Signedness.SIGNED, 2), seed=0))
    x = torch.from_numpy(datasets.uniform_images(128, 224, seed=3)).cuda()
    want = g.run(x).clone()
    for _ in range(2):
        g.autotune(x, reps=1)
        assert torch.equal(g.run(x).view(torch.int32), want.view(torch.int32))


@pytest.mark.parametrize("cand", [5, 14, 22, 31])
def test_sweep_candidate_networks_vs_oracle(cand):
    """Config 4: a ResNet-62 built on a sweep candidate table (truncated / error-injected, both
    signedness) gives the oracle graph's logits bit for bit (2 CIFAR-shaped images)."""
    torch = _torch()
    from bench import oracle_nodes, sweep_luts
    from paper_2002_09481_b200 import resnet
    from paper_2002_09481_b200.datasets import synthetic_cifar10
    from paper_2002_09481_b200.graph import GpuGraph

    nodes = resnet.cifar_resnet(10, sweep_luts()[cand], seed=0)
    x, _ = synthetic_cifar10(2, seed=77)
    want = O.run_graph(oracle_nodes(nodes), x)
    got = GpuGraph(nodes).run(torch.from_numpy(x).cuda()).cpu().numpy()
    assert bits_equal(got, want)


@pytest.mark.parametrize("c", [1024, 2048])
def test_wide_channel_quantize_and_lut_kernel_pixsum(c):
    """c = 1024 / 2048 inputs (ResNet-50 stage 3/4): the 16-channel-chunk quantizer with atomic
    per-pixel sums, read by the b-major LUT kernel (K > 512 -> sums gathered in the epilogue), and
    the ftable path -- both equal to the oracle bit for bit."""
    rng = np.random.default_rng(c)
    case = dict(x=np.maximum(rng.standard_normal((2, 5, 4, c)), 0).astype(np.float32),
                f=(rng.standard_normal((1, 1, c, 24)) * 0.05).astype(np.float32), lut=O.random_lut(rng, O.SIGNED),
                mode=O.SIGNED, padding="same", strides=(1, 1), dilations=(1, 1), accumulator=O.EXACT64,
                round_mode=O.HALF_AWAY)
    case.update(in_range=(float(case["x"].min()), float(case["x"].max())),
                f_range=(float(case["f"].min()), float(case["f"].max())))
    want, want_acc = oracle_conv(case, return_acc=True)
    for use_ft in (False, True):
        y, acc, kern = gpu_conv(case, use_ftable=use_ft)
        assert bits_equal(y, want), kern
        assert np.array_equal(acc, want_acc), kern


@pytest.mark.parametrize("kind", ["MaxPool", "AvgPool"])
@pytest.mark.parametrize("c", [3, 16, 64])
def test_pools_match_oracle(kind, c):
    """MaxPool / AvgPool (graph.py:182-199) through the executor vs the oracle, bit for bit: valid and
    explicit/same padding, strided and global windows, NaN and inf inputs (c % 4 == 0 takes the
    vectorised kernel, c = 3 the scalar one), windows of -0.0 only."""
    torch = _torch()
    from paper_2002_09481_b200.graph import GpuGraph

    rng = np.random.default_rng(c)
    x = rng.standard_normal((3, 9, 11, c)).astype(np.float32)
    x[0, 1, 2, 0] = np.nan
    x[1, 4, 4, c - 1] = np.inf
    x[2, 8, 10, 0] = -np.inf
    x[1, 0:3, 0:3, :] = -0.0  # an all -0.0 window: nansum starts from +0.0 (numpy), so AvgPool gives +0.0
    for attrs in ({"pool": [3, 3], "strides": [2, 2], "padding": "same"},
                  {"pool": [2, 2], "strides": [2, 2], "padding": "valid"},
                  {"pool": [3, 2], "strides": [1, 2], "padding": [1, 0, 1, 1]},
                  {"pool": [9, 11], "strides": [9, 11], "padding": "valid"}):
        nodes = [{"id": "in", "kind": "Input", "inputs": [], "attrs": {}},
                 {"id": "p", "kind": kind, "inputs": ["in"], "attrs": dict(attrs)}]
        got = GpuGraph(nodes).run(torch.from_numpy(x).cuda(), check=False).cpu().numpy()
        want = O.pool2d(x, attrs, kind == "MaxPool")
        assert bits_equal(got, want), (kind, c, attrs)


@pytest.mark.parametrize("mode", [O.SIGNED, O.UNSIGNED])
def test_ftable_kernel_long_k_packed_sums_exact(mode):
    """K = 3*3*2048 = 18,432 taps with full-range random 16-bit products: the packed-pair sums
    (sum of high halves up to 1.2e9) and the epilogue stay exact on every ftable variant."""
    from paper_2002_09481_b200 import _lib

    rng = np.random.default_rng(18432 + (mode == O.SIGNED))
    case = dict(x=rng.uniform(-1, 3, (1, 3, 4, 2048)).astype(np.float32),
                f=rng.standard_normal((3, 3, 2048, 20)).astype(np.float32), lut=O.random_lut(rng, mode),
                mode=mode, padding="same", strides=(1, 1), dilations=(1, 1), accumulator=O.WRAP32,
                round_mode=O.HALF_EVEN)
    case.update(in_range=(float(case["x"].min()), float(case["x"].max())),
                f_range=(float(case["f"].min()), float(case["f"].max())))
    want, want_acc = oracle_conv(case, return_acc=True)
    lib = _lib.load()
    kpad = 3 * 3 * 2048
    for v in range(1, lib.axb_ft_variant_count()):
        if 32 % LAYOUT_BLOCK[lib.axb_ft_variant_layout(v)]:  # 64-channel blocks: cout 20 pads to 32
            continue
        if kpad > lib.axb_ft_variant_max_k(v):  # CX variants: 32-bit epilogue, K <= 8192 (layout_ok)
            with pytest.raises(ValueError, match="K > 8192"):
                gpu_conv(case, ft_variant=v)
            continue
        y, acc, kern = gpu_conv(case, ft_variant=v)
        assert kern.startswith(("ft", "cm", "c32", "c16")), kern
        assert bits_equal(y, want), kern
        assert np.array_equal(acc, want_acc), kern


def test_run_benchmark_report_and_outputs(tmp_path):
    """benchmark.run_benchmark (reference bench.py:37-87 on the GPU engine): outputs bit-identical to the
    reference executor's for a reference model file; report phases partition t_init + t_comp; MAC count
    = graph MACs x images; CIFAR-10 files run through the on-device record decode."""
    from paper_2002_09481_b200 import formats as F
    from paper_2002_09481_b200 import resnet
    from paper_2002_09481_b200 import types as T
    from paper_2002_09481_b200.benchmark import run_benchmark, speedup
    from paper_2002_09481_b200.datasets import synthetic_cifar10

    g = load_golden("formats")
    (tmp_path / "ax.json").write_bytes(g["model_json"].tobytes())
    (tmp_path / "ax.weights.bin").write_bytes(g["model_weights"].tobytes())
    F.save_lut(T.truncated_lut(T.Signedness.SIGNED, 2), tmp_path / "ax.axm")
    x = g["model_input"]
    # one range-batch = the reference executor's batch (ranges are per batch, graph.py:270-275)
    report, out = run_benchmark(tmp_path / "ax.json", x, batch_size=x.shape[0])
    assert bits_equal(out, g["model_logits"])
    assert report.t_init > 0 and report.t_comp > 0 and report.phase_seconds["lut_lookup"] > 0
    assert abs(sum(report.phase_seconds.values()) - report.total) <= 1e-9 * max(1.0, report.total)
    assert report.mac_count > 0 and report.per_layer
    F.save_report(report, tmp_path / "r.json")
    back = F.load_report(tmp_path / "r.json")
    assert back.mac_count == report.mac_count and back.phase_seconds == report.phase_seconds
    assert F.report_csv(back).startswith("name,seconds,percent\nlut_lookup,")
    assert speedup(report, report) == 1.0

    lut = T.truncated_lut(T.Signedness.SIGNED, 2)
    nodes = resnet.cifar_resnet(1, lut, seed=0)
    imgs, labels = synthetic_cifar10(200, seed=5)
    F.save_cifar10(tmp_path / "data.bin", imgs, labels)
    rep_f, out_f = run_benchmark(nodes, tmp_path / "data.bin", batch_size=64)
    rep_a, out_a = run_benchmark(nodes, imgs, batch_size=64, batches=4)
    assert out_f.shape[0] == 200 and bits_equal(out_f, out_a)
    assert rep_f.mac_count == rep_a.mac_count == 200 * _graph_macs(nodes)


def _graph_macs(nodes):
    from oracle.axemu_oracle import graph_mac_count

    return graph_mac_count(nodes, (1, 32, 32, 3))


def test_projection_reads_first_conv_codes():
    """A ResNet projection (1x1, unpadded, same input as the block's first conv) reads that conv's
    zp-padded code tensor instead of quantizing again: one quantize launch fewer per projection, and
    the logits stay bit-identical to the reference executor's (the projections host the fused
    residual Add + ReLU, so their own values are covered through the logits)."""
    torch = _torch()
    from paper_2002_09481_b200 import resnet
    from paper_2002_09481_b200 import types as T
    from paper_2002_09481_b200.graph import GpuGraph

    g = load_golden("nets")
    gg = GpuGraph(resnet.cifar_resnet(1, T.truncated_lut(T.Signedness.SIGNED, 2), seed=0))
    y = gg.run(torch.from_numpy(g["r8_trunc2_x"]).cuda()).cpu().numpy()
    shared = {nid: p.share_from for nid, p in gg.conv_plans.items() if p.share_from}
    assert shared == {"s1b0.proj": "s1b0.a", "s2b0.proj": "s2b0.a"}, shared
    assert bits_equal(y, g["r8_trunc2_logits"])
    prof = []
    gg.run(torch.from_numpy(g["r8_trunc2_x"]).cuda(), profile=prof)
    assert gg.launches == 1 + 10 + 10 - 2 + 1  # input range, 10 convs, 10 quantizes minus 2 shared, pool


# axb_ft_variant_layout -> channel block of the table the variant reads (0: pair-major, 16-channel tiles)
LAYOUT_BLOCK = {0: 16, 1: 32, 2: 64, 3: 32, 4: 16}


@pytest.mark.parametrize("layout", [1, 2, 3, 4])
@pytest.mark.parametrize("mode", [O.SIGNED, O.UNSIGNED])
def test_code_major_variants_vs_oracle(mode, layout):
    """The code-major kernel families -- cm32_* (32-channel blocks, LDS.128 of 4 pairs, layout 1) and the
    CX family c64_* / c32_* / c16_* (64 / 32 / 16-channel blocks in 128-byte rows, one pixel per quarter /
    eighth / sixteenth of a warp instruction, layouts 2 / 3 / 4) -- over shapes the pair-major test does
    not reach: cout 16 / 32 / 64 / 96 / 128 / 192 (one to many channel blocks, ragged 61 and 150), wide and
    odd input channels, stride 2, dilation 2, ragged pixel tiles, every accumulator mode, K = 4608, and
    tiles cut by the tail split (more CTAs than tiles)."""
    from paper_2002_09481_b200 import _lib

    lib = _lib.load()
    cms = [v for v in range(1, lib.axb_ft_variant_count()) if lib.axb_ft_variant_layout(v) == layout]
    assert len(cms) >= 2
    blk = LAYOUT_BLOCK[layout]
    rng = np.random.default_rng(4096 + (mode == O.SIGNED))
    shapes = [((3, 9, 13, 16), (3, 3, 16, 32), (1, 1), (1, 1), "same", O.EXACT64),
              ((2, 11, 10, 48), (3, 3, 48, 64), (2, 2), (1, 1), "same", O.WRAP32),
              ((2, 12, 12, 64), (1, 1, 64, 96), (1, 1), (1, 1), "valid", O.SATURATE32),
              ((1, 14, 9, 37), (3, 3, 37, 61), (1, 2), (2, 2), "same", O.EXACT64),
              ((3, 17, 15, 32), (3, 3, 32, 128), (1, 1), (1, 1), "same", O.EXACT64),
              ((2, 9, 9, 80), (1, 1, 80, 150), (2, 2), (1, 1), "valid", O.WRAP32),
              ((1, 5, 6, 512), (3, 3, 512, 192), (1, 1), (1, 1), "same", O.EXACT64),
              ((4, 16, 16, 3), (3, 3, 3, 16), (1, 1), (1, 1), "same", O.EXACT64),
              ((2, 19, 21, 16), (3, 3, 16, 48), (2, 1), (1, 1), "same", O.EXACT64)]
    for xs, fs, st, dil, pad, acc in shapes:
        if -(-fs[3] // 16) * 16 % blk:
            continue
        x = np.maximum(rng.standard_normal(xs), 0).astype(np.float32) if acc != O.WRAP32 else \
            rng.uniform(-2, 3, xs).astype(np.float32)
        case = dict(x=x, f=rng.standard_normal(fs).astype(np.float32), lut=O.random_lut(rng, mode), mode=mode,
                    padding=pad, strides=st, dilations=dil, accumulator=acc, round_mode=O.HALF_EVEN)
        case.update(in_range=(float(x.min()), float(x.max())),
                    f_range=(float(case["f"].min()), float(case["f"].max())))
        want, want_acc = oracle_conv(case, return_acc=True)
        for v in cms:
            y, acc_got, kern = gpu_conv(case, ft_variant=v)
            assert kern.startswith("cm32" if layout == 1 else f"c{blk}"), kern
            assert bits_equal(y, want), (kern, xs, fs)
            assert np.array_equal(acc_got, want_acc), (kern, xs, fs)


def test_graph_forced_code_major_matches_reference():
    """Every ResNet-8 layer with 32-channel blocks forced onto each code-major variant (fused bias,
    residual, ReLU, next-layer range in its epilogue; projections reading shared codes): logits
    bit-identical to the reference executor's golden logits."""
    torch = _torch()
    from paper_2002_09481_b200 import _lib, resnet
    from paper_2002_09481_b200 import types as T
    from paper_2002_09481_b200.graph import GpuGraph

    lib = _lib.load()
    g = load_golden("nets")
    gg = GpuGraph(resnet.cifar_resnet(1, T.truncated_lut(T.Signedness.SIGNED, 2), seed=0))
    x = torch.from_numpy(g["r8_trunc2_x"]).cuda()
    gg.run(x)
    for v in [v for v in range(1, lib.axb_ft_variant_count()) if lib.axb_ft_variant_layout(v) == 1]:
        picks = {nid: (v if p.layer.cm_ok else 0) for nid, p in gg.conv_plans.items()}
        assert sum(1 for p in picks.values() if p) >= 5, picks
        gg.set_tuning(picks)
        prof = []
        y = gg.run(x, profile=prof).cpu().numpy()
        assert sum(1 for *_, fam in prof if fam == "lutconv_ftcm") == sum(1 for p in picks.values() if p)
        assert bits_equal(y, g["r8_trunc2_logits"]), lib.axb_ft_variant_name(v)


def test_graph_rejects_range_nodes_over_another_tensor():
    """An AxConv2D whose Min/Max inputs range over a different tensor than its data input (the reference
    would quantize with that other range, graph.py:248-251) is refused at planning time instead of
    silently quantizing with the data input's range slot."""
    from paper_2002_09481_b200.graph import GpuGraph

    f = np.ones((1, 1, 3, 4), np.float32)
    conv = {"filters": f, "strides": (1, 1), "dilations": (1, 1), "padding": "valid", "f_min": 0.0, "f_max": 1.0,
            "lut": _lut(O.exact_lut(O.SIGNED), O.SIGNED)}
    base = [{"id": "in", "kind": "Input", "inputs": [], "attrs": {}},
            {"id": "r", "kind": "ReLU", "inputs": ["in"], "attrs": {}}]
    bad = base + [{"id": "lo", "kind": "Min", "inputs": ["r"], "attrs": {}},
                  {"id": "hi", "kind": "Max", "inputs": ["r"], "attrs": {}},
                  {"id": "c", "kind": "AxConv2D", "inputs": ["in", "lo", "hi"], "attrs": conv}]
    with pytest.raises(ValueError, match="range input"):
        GpuGraph(bad)
    swapped = base + [{"id": "lo", "kind": "Min", "inputs": ["in"], "attrs": {}},
                      {"id": "hi", "kind": "Max", "inputs": ["in"], "attrs": {}},
                      {"id": "c", "kind": "AxConv2D", "inputs": ["in", "hi", "lo"], "attrs": conv}]
    with pytest.raises(ValueError, match="must be a Min node"):
        GpuGraph(swapped)
    good = base + [{"id": "lo", "kind": "Min", "inputs": ["in"], "attrs": {}},
                   {"id": "hi", "kind": "Max", "inputs": ["in"], "attrs": {}},
                   {"id": "c", "kind": "AxConv2D", "inputs": ["in", "lo", "hi"], "attrs": conv}]
    GpuGraph(good)


def test_graph_frees_intermediates_after_last_reader():
    """Activations are released after their last executed reader (fused Add/ReLU and Min/Max nodes read
    nothing at run time): ResNet-50 at 64 images peaks well below the sum of all its activations."""
    torch = _torch()
    from paper_2002_09481_b200.graph import GpuGraph

    nodes, x = _bench_config("r50")
    gg = GpuGraph(nodes)
    xd = torch.from_numpy(x[:64]).cuda()
    gg.run(xd)
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    trace = {}
    gg.run(xd, trace=trace)  # trace keeps every node's value alive
    torch.cuda.synchronize()
    keep_all = torch.cuda.max_memory_allocated() - base
    del trace
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    gg.run(xd)
    torch.cuda.synchronize()
    freed = torch.cuda.max_memory_allocated() - base
    assert freed < 0.35 * keep_all, (freed, keep_all)


def _ord2f(i: int) -> float:
    b = i if i >= 0 else i ^ 0x7FFFFFFF
    return float(np.array([b], np.int32).view(np.float32)[0])


@pytest.mark.gpu
@pytest.mark.parametrize("bad", [None, np.nan, np.inf, -np.inf])
@pytest.mark.parametrize("relu", [False, True])
def test_cx_output_range_and_nonfinite_flag(bad, relu):
    """The CX epilogue's fused next-layer range (graph.py:270-275 over the conv output) is the exact
    min/max of what it stored, and a non-finite output (here from the residual Add, graph.py:282-286)
    raises AXB_FLAG_OUT_NONFINITE -- for every CX variant, ragged tiles and the tail split included."""
    torch = _torch()
    from paper_2002_09481_b200 import _lib
    from paper_2002_09481_b200 import types as T
    from paper_2002_09481_b200.layer import ConvLayer

    lib = _lib.load()
    rng = np.random.default_rng(11)
    x = torch.relu(torch.from_numpy(rng.standard_normal((2, 9, 11, 32)).astype(np.float32))).cuda()
    f = (rng.standard_normal((3, 3, 32, 64)) * 0.05).astype(np.float32)
    lay = ConvLayer(f, (float(f.min()), float(f.max())), T.truncated_lut(T.Signedness.SIGNED, 2),
                    T.ConvGeometry(padding="same"),
                    bias=(rng.standard_normal(64) * 0.05).astype(np.float32))
    lay.set_input_params(0.0, float(x.max()))
    res = torch.from_numpy(rng.standard_normal((2, 9, 11, 64)).astype(np.float32))
    if bad is not None:
        res[1, 3, 4, 5] = float(bad)
    res = res.cuda()
    n = 0
    for v in range(1, lib.axb_ft_variant_count()):
        if not lib.axb_ft_variant_name(v).decode().startswith("c") or \
                64 % LAYOUT_BLOCK[lib.axb_ft_variant_layout(v)]:
            continue
        orng = torch.tensor([2**31 - 1, -2**31], dtype=torch.int32, device="cuda")
        flags = torch.zeros(2, dtype=torch.int32, device="cuda")
        y = lay.run(x, None, residual=res, relu=relu, out_range=orng.data_ptr(), out_flag=flags[0].data_ptr(),
                    quant_flag=flags[1].data_ptr(), ft_variant=v)
        torch.cuda.synchronize()
        name = lib.axb_ft_variant_name(v).decode()
        fl = int(flags[0].item())
        if bad is None or (relu and bad == -np.inf):  # ReLU after the Add: -inf -> 0, the output is finite
            assert fl & _lib.FLAG_OUT_NONFINITE == 0, name
            lo, hi = (_ord2f(int(t)) for t in orng.tolist())
            assert lo == float(y.min()) and hi == float(y.max()), name
        else:
            assert fl & _lib.FLAG_OUT_NONFINITE, name
        n += 1
    assert n >= 5


@pytest.mark.gpu
def test_quantizer_flat_path_sweep():
    """The flat quantizer (unpadded input, no per-pixel sums: what every 1x1 CX layer runs) vs
    quantize_values (quantizer.py:120-131) on dense near-tie sweeps, all modes, ragged unit tails
    (element counts not a multiple of the 512-float warp unit), host and device coefficients, and the
    non-finite flag (tensor.py:143-149 -> ValueError)."""
    torch = _torch()
    from paper_2002_09481_b200 import _lib

    lib = _lib.load()
    s = torch.cuda.current_stream().cuda_stream
    rng = np.random.default_rng(78)
    rounds = {O.HALF_AWAY: 0, O.HALF_EVEN: 1, O.TOWARD_ZERO: 2}
    for trial in range(12):
        mode = (O.SIGNED, O.UNSIGNED)[trial % 2]
        rname = list(rounds)[trial % 3]
        mn = float(-abs(rng.standard_normal()) * 10 ** rng.uniform(-3, 3)) if trial % 4 else 0.0
        mx = float(abs(rng.standard_normal()) * 10 ** rng.uniform(-3, 3))
        mn, mx = float(np.float32(mn)), float(np.float32(mx))  # a device range holds float32 extremes
        scale, zp = O.compute_coeffs(mn, mx, mode, rname)
        lo, _ = O.bounds(mode)
        k = np.arange(-300, 300, dtype=np.float64)
        base = np.concatenate([(k + 0.5 - zp + lo) * scale, (k - zp + lo) * scale]).astype(np.float32)
        near = (base.view(np.int32)[:, None] + np.arange(-3, 4, dtype=np.int32)[None, :]).reshape(-1).view(np.float32)
        vals = np.concatenate([near, rng.uniform(mn * 1.5, mx * 1.5, 70000).astype(np.float32), [mn, mx]])
        vals = vals[np.isfinite(vals)].astype(np.float32)
        hp_ = _lib.QParams()
        _lib.check(lib.axb_coeffs_host(mn, mx, int(mode == O.SIGNED), rounds[rname], hp_))
        prm = torch.zeros(_lib.QPARAMS_BYTES, dtype=torch.uint8, device="cuda")
        _lib.check(lib.axb_params_upload(hp_, prm.data_ptr(), s))
        ordr = torch.from_numpy(np.array([mn, mx], np.float32).view(np.int32)).cuda()
        ordr = torch.where(ordr >= 0, ordr, ordr ^ 0x7FFFFFFF).to(torch.int32)
        for c in (16, 64, 256):
            v = vals[: len(vals) // c * c]
            want = O.quantize_values(v, scale, zp, mode, rname)
            n = len(v) // c
            x = torch.from_numpy(v.reshape(1, 1, n, c)).cuda()
            for dev_range in (False, True):
                codes = torch.full((n * c,), 0xAB, dtype=torch.uint8, device="cuda")
                fl = torch.zeros(1, dtype=torch.int32, device="cuda")
                if dev_range:
                    p2 = torch.zeros(_lib.QPARAMS_BYTES, dtype=torch.uint8, device="cuda")
                    _lib.check(lib.axb_quantize_pad_range(x.data_ptr(), 1, 1, n, c, 0, 0, 0, 0, c, ordr.data_ptr(),
                                                          int(mode == O.SIGNED), rounds[rname], p2.data_ptr(),
                                                          codes.data_ptr(), None, fl.data_ptr(), s))
                else:
                    _lib.check(lib.axb_quantize_pad(x.data_ptr(), 1, 1, n, c, 0, 0, 0, 0, c, prm.data_ptr(),
                                                    int(mode == O.SIGNED), rounds[rname], codes.data_ptr(), None,
                                                    fl.data_ptr(), s))
                got = codes.cpu().numpy().view(np.int8 if mode == O.SIGNED else np.uint8)
                assert np.array_equal(got, want), (trial, c, dev_range, np.flatnonzero(got != want)[:5])
                assert int(fl.item()) == 0
    # non-finite input -> FLAG_NONFINITE
    for bad in (np.nan, np.inf, -np.inf):
        v = rng.standard_normal(4096 * 16).astype(np.float32)
        v[777] = bad
        x = torch.from_numpy(v.reshape(1, 1, 4096, 16)).cuda()
        codes = torch.empty(v.size, dtype=torch.uint8, device="cuda")
        fl = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.check(lib.axb_quantize_pad(x.data_ptr(), 1, 1, 4096, 16, 0, 0, 0, 0, 16, prm.data_ptr(), 1, 1,
                                        codes.data_ptr(), None, fl.data_ptr(), s))
        assert int(fl.item()) & _lib.FLAG_NONFINITE, bad
