#!/usr/bin/env python
"""Benchmark: approximate-LUT ResNet inference on B200 (one process per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload r50|r8|r62|r62sweep|mbv1]
                    [--impl b200|reference] [--stub]

A step = one range-batch of synthetic images through the whole transformed
ResNet graph (every conv an AxConv2D with the approximate truth table, the
classifier a 1x1 AxConv2D): range reduction, quantize + zp-pad, LUT implicit
GEMM with fused correction/dequant/bias/residual/ReLU/next-range epilogue,
pools.  Default workload = the north-star target, BASELINE configs[2]:
ResNet-50 224x224, batch 256 per GPU, truncated_lut(signed, 2), calibrated
weights (resnet.py).

``--gpus N`` without a torch.distributed environment re-launches this script
under ``python -m torch.distributed.run`` with N local ranks (127.0.0.1, NCCL,
``NCCL_DEBUG=INFO`` limited to the INIT subsystem so every rank prints its
communicator line).  Launched by torchrun directly, it uses the environment's
ranks.  Sharding: range-batches (ranges are per batch,
graph.py:270-275) -- every rank runs its own batch, zero per-layer
communication ("scaling": "weak"); config 4 (``r62sweep``) -- the 32 candidate
tables are dealt round-robin, uneven counts allowed ("scaling": "strong").
NCCL only all-gathers logits and all-reduces prediction counts and device
times after the timed region.

Timing: W warm-up steps, then K steps bracketed by barrier + synchronize; each
step is timed with CUDA events on the launching stream and L2 is flushed
(256 MiB write) between steps outside the events; the job time is the max
over ranks.  value = approximate GMAC/s of the whole job (algorithmic MACs as
graph_mac_count, graph.py:316-349); images/s alongside.  e2e = the same metric
through the public GpuGraph.run_pipelined API from pinned HOST batches, H2D
of the inputs and D2H of the logits inside the timed region.  After the timed
region rank 0's logits are compared bit-for-bit (sha256) with the real
reference's output for the same batch (tests/golden/bench.npz): "parity".

--impl reference: the reference's CPU algorithm on the host cores (the pinned
oracle port: numpy + C/OpenMP LUT-GEMM, all host threads; plus the real numba
``axemu`` package from baseline/_ref when present) on bounded samples of the
same workload, rank 0 only.

--stub: the launcher / sharding / gather / JSON path on CPU with gloo and a
synthetic step (no GPU) -- what the CPU tests exercise.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "approximate GMAC/s and images/s (ResNet, synthetic) at 1/2/4/8 B200 vs CPU ref"
# paper-derived GTX 1080 approximate throughput for the same CIFAR nets
PAPER_GMACS = {"r8": 140.0, "r62": 95.5}
BENCH_SEED = 1000  # rank r's range-batch is seeded BENCH_SEED + r (tests/golden/make_golden.py)


def workload_spec(name: str, lut_kind: str):
    from paper_2002_09481_b200 import resnet
    from paper_2002_09481_b200 import types as T

    if lut_kind == "trunc2":
        lut = T.truncated_lut(T.Signedness.SIGNED, 2)
        lut_desc = "truncated_lut(signed, 2)"
    elif lut_kind == "exact":
        lut = T.exact_lut(T.Signedness.SIGNED)
        lut_desc = "exact_lut(signed)"
    else:
        lut = T.random_lut(np.random.default_rng(123), T.Signedness.SIGNED)
        lut_desc = "random_lut(signed, seed 123)"
    if name == "r8":
        return dict(nodes=resnet.cifar_resnet(1, lut, seed=0), batch=1024, kind="cifar", lut=lut_desc,
                    desc="ResNet-8 CIFAR-10 (He 6n+2, n=1; 9 convs + 1x1 AxConv2D classifier), calibrated")
    if name == "r62":
        return dict(nodes=resnet.cifar_resnet(10, lut, seed=0), batch=1000, kind="cifar", lut=lut_desc,
                    desc="ResNet-62 CIFAR-10 (He 6n+2, n=10; 63 convs + 1x1 AxConv2D classifier), calibrated")
    if name == "r50":
        return dict(nodes=resnet.resnet50(lut, seed=0), batch=256, kind="imagenet", lut=lut_desc,
                    desc="ResNet-50 v1.5 224x224 (53 convs + 1x1 AxConv2D classifier), BN folded, calibrated")
    if name == "mbv1":
        return dict(nodes=resnet.mobilenet_v1(lut, seed=0), batch=256, kind="imagenet", lut=lut_desc,
                    desc="MobileNet-v1-shaped 224x224 (stem + 13 x (depthwise 3x3 + pointwise 1x1) + 1x1 AxConv2D "
                         "classifier; config 5 depthwise approximate conv), BN folded, calibrated")
    if name == "r62sweep":
        return dict(nodes=resnet.cifar_resnet(10, sweep_luts()[0], seed=0), batch=1000, kind="cifar",
                    lut="32 candidates: truncated_lut(mode, d) d=0..7 x {signed, unsigned} + 16 perturbed_lut "
                        "(exact + uniform error of 2..256, both signedness)",
                    desc="ResNet-62 CIFAR-10 multiplier sweep over 32 candidate tables (config 4), calibrated",
                    sweep=True)
    raise SystemExit(f"unknown workload {name}")


def lib_variant_name(v: int) -> str:
    from paper_2002_09481_b200.graph import variant_name

    return variant_name(int(v))


def sweep_luts():
    """Config 4's 32 candidate multipliers."""
    from paper_2002_09481_b200 import types as T

    # 16 truncated multipliers + 16 error-injected ones (uniform random tables, as in the reference's
    # test helper, drive a 63-conv network to non-finite activations -> ValueError, graph.py:273-274)
    luts = [T.truncated_lut(m, d) for m in (T.Signedness.SIGNED, T.Signedness.UNSIGNED) for d in range(8)]
    luts += [T.perturbed_lut(np.random.default_rng(5000 + i), T.Signedness.SIGNED if i % 2 else T.Signedness.UNSIGNED,
                             1 + i // 2) for i in range(16)]
    return luts


def units_of(spec, world: int, rank: int) -> list[int]:
    """This rank's networks: [0] (its own range-batch) or its round-robin share of the 32 tables."""
    from paper_2002_09481_b200.dist import shard

    return shard(len(sweep_luts()), world, rank) if spec.get("sweep") else [0]


def make_images(kind: str, n: int, seed: int):
    from paper_2002_09481_b200 import datasets

    if kind == "cifar":
        return datasets.synthetic_cifar10(n, seed=seed)
    return datasets.synthetic_imagenet(n, seed=seed)


def make_config(spec, args, batch: int, world: int, macs_img: int) -> dict:
    """The workload description shared by both arms (same dict -> same config)."""
    return {"workload": spec["desc"], "batch_per_gpu": batch, "lut": spec["lut"],
            "networks": 32 if spec.get("sweep") else 1, "macs_per_image": macs_img,
            "images": f"synthetic_{'cifar10' if spec['kind'] == 'cifar' else 'imagenet'}(batch, seed="
                      f"{BENCH_SEED} + rank)" if not spec.get("sweep") else
                      f"synthetic_cifar10(batch, seed={BENCH_SEED}), every candidate table",
            "parallelism": (f"dp{world} (candidate tables sharded round-robin)" if spec.get("sweep")
                            else f"dp{world} (one range-batch per GPU)"),
            "l2": "flushed between timed steps (256 MiB write, outside the events)"}


# ---------------------------------------------------------------------------- launcher


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_ranks(args, argv) -> int:
    """Re-run this script under torch.distributed.run with ``args.gpus`` local ranks."""
    if not args.stub and not args.share_device:
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but only {have} visible CUDA "
                                                         "devices"}), flush=True)
            return 1
    env = dict(os.environ)
    # every rank prints its communicator line (ncclCommInitRankConfig ... nranks N); a box-level NCCL_DEBUG
    # (seen: one that printed only the version line) would hide it
    env["NCCL_DEBUG"] = "INFO"
    env["NCCL_DEBUG_SUBSYS"] = "INIT"
    env.setdefault("OMP_NUM_THREADS", "4")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(Path(__file__).resolve()), *argv]
    print("[bench] launching:", " ".join(cmd), file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


# ---------------------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi clocks + throttle reasons, sampled every 20 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        if not self.lines:  # timed region shorter than one sampling period: take one sample now
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=20)
                self.lines.extend(out.stdout.strip().splitlines())
            except Exception:
                pass
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------- CPU baselines


def oracle_nodes(nodes):
    out = []
    for n in nodes:
        a = dict(n["attrs"])
        if "lut" in a:
            a["mode"], a["lut"] = a["lut"].mode.value, a["lut"].entries
        out.append({"id": n["id"], "kind": n["kind"], "inputs": n["inputs"], "attrs": a})
    return out


def cpu_reference_rate(spec, macs_per_img: int, budget_s: float, seed: int = 0, warm: bool = True):
    """Time the oracle port (reference algorithm, all host threads) on a bounded sample."""
    from oracle import axemu_oracle as O

    onodes = oracle_nodes(spec["nodes"])
    n = 2 if spec["kind"] == "imagenet" else 16
    x, _ = make_images(spec["kind"], n, seed)
    if warm:
        O.run_graph(onodes, x[:1])  # warm-up (page-in, OpenMP pool)
    t0 = time.perf_counter()
    O.run_graph(onodes, x)
    dt = time.perf_counter() - t0
    # scale the sample towards the time budget (bounded)
    scale = max(1, min(int(budget_s / max(dt, 1e-3)), 64 if spec["kind"] == "cifar" else 8))
    if scale > 1:
        n2 = n * scale
        x, _ = make_images(spec["kind"], n2, seed)
        t0 = time.perf_counter()
        O.run_graph(onodes, x)
        dt = time.perf_counter() - t0
        n = n2
    gmacs = n * macs_per_img / dt / 1e9
    return dict(value=round(gmacs, 4), unit="GMAC/s", images_per_s=round(n / dt, 3), cores=O.threads(),
                kind="port", images=n, seconds=round(dt, 3),
                sample=f"{n} images of the same workload through the oracle port "
                       f"(numpy + C/OpenMP int64 LUT-GEMM), {dt:.2f} s")


def reference_numba_rate(spec, macs_per_img: int, budget_s: float, seed: int = 0):
    """The real reference package (axemu, numba ``gemm`` engine, all host threads) from baseline/_ref,
    if it was installed there; None otherwise."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "axemu").is_dir():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/axemu_numba_cache")
    sys.path.insert(0, str(ref))
    try:
        import numba
        import axemu
        from axemu import LayerGraph, Layout, MultLut, Node, NodeKind, Signedness, Tensor4
    except Exception as e:  # pragma: no cover - depends on the box
        return {"unavailable": f"import failed: {e}"}
    ref_nodes = []
    for nd in spec["nodes"]:
        a = dict(nd["attrs"])
        if "lut" in a:
            a["lut"] = MultLut(Signedness(a["lut"].mode.value), a["lut"].entries)
        ref_nodes.append(Node(nd["id"], NodeKind(nd["kind"]), list(nd["inputs"]), a))
    g = LayerGraph(ref_nodes)
    n = 2 if spec["kind"] == "imagenet" else 16
    x, _ = make_images(spec["kind"], n, seed)
    t0 = time.perf_counter()
    axemu.run(g, Tensor4(x[:1], Layout.NHWC), "gemm")  # warm-up: numba JIT (cached under NUMBA_CACHE_DIR)
    t_init = time.perf_counter() - t0
    t0 = time.perf_counter()
    axemu.run(g, Tensor4(x, Layout.NHWC), "gemm")
    dt = time.perf_counter() - t0
    scale = max(1, min(int(budget_s / max(dt, 1e-3)), 64 if spec["kind"] == "cifar" else 4))
    if scale > 1:
        n *= scale
        x, _ = make_images(spec["kind"], n, seed)
        t0 = time.perf_counter()
        axemu.run(g, Tensor4(x, Layout.NHWC), "gemm")
        dt = time.perf_counter() - t0
    return dict(value=round(n * macs_per_img / dt / 1e9, 4), unit="GMAC/s", images_per_s=round(n / dt, 3),
                cores=int(numba.config.NUMBA_NUM_THREADS), kind="reference", t_init_s=round(t_init, 2),
                sample=f"{n} images through the real axemu.graph.run(engine='gemm') (numba, baseline/_ref), "
                       f"{dt:.2f} s after a 1-image warm-up")


def reference_arm(args, spec, batch, world, rank, macs_img):
    """--impl reference: the reference's CPU implementation on the host cores, rank 0 only."""
    if rank != 0:
        return
    from oracle import axemu_oracle as O

    onodes = oracle_nodes(spec["nodes"])
    xw, _ = make_images(spec["kind"], 1, 999)
    for _ in range(args.warmup):  # W real warm-up passes (page-in, OpenMP pool) on a 1-image sample
        O.run_graph(onodes, xw)
    imgs = secs = 0.0
    info = None
    for k in range(max(1, args.steps)):
        info = cpu_reference_rate(spec, macs_img, budget_s=min(args.cpu_budget, 20.0) / max(1, args.steps) * 2,
                                  seed=k, warm=False)
        imgs += info["images"]
        secs += info["seconds"]
    val = round(imgs * macs_img / secs / 1e9, 4)
    numba_rate = None if args.no_numba else reference_numba_rate(spec, macs_img, budget_s=min(args.cpu_budget, 10))
    cpu = {"value": val, "unit": "GMAC/s", "cores": info["cores"], "kind": "port",
           "sample": f"{int(imgs)} images in {args.steps} steps of the same workload through the oracle port "
                     f"(numpy + C/OpenMP int64 LUT-GEMM), {secs:.2f} s"}
    if numba_rate is not None:
        cpu["reference_numba"] = numba_rate
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "GMAC/s",
            "images_per_s": round(imgs / secs, 3), "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(secs * 1e3 / max(1, args.steps), 3), "higher_is_better": True,
            "scaling": "strong" if spec.get("sweep") else "weak", "vs_baseline": None,
            "dtype": "u8", "data": "synthetic",
            "config": make_config(spec, args, batch, world, macs_img),
            "cpu_baseline": cpu,
            "e2e": {"value": val, "unit": "GMAC/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- one rank's work


class CpuEvent:
    """torch.cuda.Event stand-in for --stub (host clock)."""

    def __init__(self, enable_timing=True):
        self.t = None

    def record(self, stream=None):
        self.t = time.perf_counter()

    def elapsed_time(self, other) -> float:
        return (other.t - self.t) * 1e3


def stub_rank(args, spec, batch, ctx, units) -> dict:
    """Synthetic step on the host: deterministic logits per (table, image), ~2 ms per network."""
    classes = 10 if spec["kind"] == "cifar" else 1000
    rng_seed = BENCH_SEED if spec.get("sweep") else BENCH_SEED + ctx["rank"]

    def step():
        ys = []
        for u in units:
            r = np.random.default_rng([rng_seed, u])
            ys.append(r.standard_normal((batch, classes)).astype(np.float32))
            time.sleep(0.002)
        return np.stack(ys) if ys else np.zeros((0, batch, classes), np.float32)

    for _ in range(args.warmup):
        step()
    ctx["barrier"]()
    evs = []
    for _ in range(args.steps):
        e0, e1 = CpuEvent(), CpuEvent()
        e0.record()
        y = step()
        e1.record()
        evs.append((e0, e1))
    ctx["barrier"]()
    total_ms = sum(a.elapsed_time(b) for a, b in evs)
    _, labels = make_images(spec["kind"], batch, rng_seed) if spec["kind"] == "cifar" else (None, np.zeros(batch))
    return {"total_ms": total_ms, "e2e_ms": total_ms, "conv_ms": 0.0, "logits": y, "labels": labels,
            "launches": 0, "extra": {}}


def device_rank(args, spec, batch, ctx, units) -> dict:
    import torch

    from paper_2002_09481_b200 import resnet
    from paper_2002_09481_b200.graph import GpuGraph

    dev = ctx["device"]
    local = dev.index
    if spec.get("sweep"):
        luts = sweep_luts()
        graphs = [GpuGraph(resnet.cifar_resnet(10, luts[i], seed=0), device=local) for i in units]
    else:
        graphs = [GpuGraph(spec["nodes"], device=local)]
    seed = BENCH_SEED if spec.get("sweep") else BENCH_SEED + ctx["rank"]
    imgs, labels = make_images(spec["kind"], batch, seed=seed)
    x_dev = torch.from_numpy(imgs).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    barrier = ctx["barrier"]

    def run_all(x, check=False, profile=None, mprofile=None):
        return [g.run(x, check=check, profile=profile, mprofile=mprofile) for g in graphs]

    # warm-up (also prepares filters once: hoisted quantize_filters), per-layer kernel autotune on the
    # first batch (outside the timed region; bit-identity of all variants checked), CUDA-graph capture
    tuned = {}
    if graphs and args.tuned_from:  # replay an earlier run's picks (e.g. under ncu, whose replays distort
        # timing) from the first warm-up on, so a launch list / traffic capture sees only the tuned kernels
        graphs[0].set_tuning(json.loads(Path(args.tuned_from).read_text()))
        tuned = {"from": args.tuned_from}
    for _ in range(args.warmup):
        run_all(x_dev, check=True)
    if graphs:
        if not args.tuned_from and not args.no_autotune:
            tuned = graphs[0].autotune(x_dev)
            if args.tuned_out:
                Path(args.tuned_out).write_text(json.dumps(graphs[0].tuning_names()))
        for g in graphs[1:]:  # same architecture (sweep candidates): same shapes -> same picks
            if tuned:
                g.copy_tuning(graphs[0])
    torch.cuda.synchronize()
    run_all(x_dev)
    launches = sum(g.launches for g in graphs)
    for g in graphs:
        g.capture(tuple(x_dev.shape))
    for _ in range(args.warmup):
        ys = [g.replay(x_dev) for g in graphs]
    torch.cuda.synchronize()

    # ------------------------------------------------ device-resident timed region (graph replay)
    sampler = ClockSampler(local)
    sampler.start()
    barrier()
    step_ev = []
    for _ in range(args.steps):
        flush.zero_()  # write > L2 (126 MB) between timed steps
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ys = [g.replay(x_dev, check=False) for g in graphs]
        e1.record()
        step_ev.append((e0, e1))
    barrier()
    clocks = sampler.stop()
    total_ms = sum(a.elapsed_time(b) for a, b in step_ev)
    for g in graphs:
        g.check_flags()
    y = torch.stack([t.reshape(batch, -1) for t in ys]) if ys else torch.zeros((0, batch, 1), device=dev)

    # ------------------------------------------------ per-kernel times (eager pass, events per launch)
    profile: list = []
    mprofile: list = []
    barrier()
    for _ in range(args.steps):
        flush.zero_()
        run_all(x_dev, profile=profile, mprofile=mprofile)
    barrier()
    torch.cuda.synchronize()

    # ------------------------------------------------ end-to-end through the public API (host buffers)
    # GpuGraph.run_pipelined: pinned host batch -> H2D (copy stream, overlapping the previous step's
    # compute) -> captured step -> D2H of the logits (+ flags); L2 flushed before each step.  CIFAR
    # workloads ship the CIFAR-10 binary records (the reference's on-disk input, formats.py:131-171),
    # decoded on the device inside the captured step; ImageNet-shaped workloads ship fp32 NHWC images.
    if spec["kind"] == "cifar":
        from paper_2002_09481_b200.formats import encode_cifar10

        host_np = encode_cifar10(imgs, labels)
    else:
        host_np = imgs
    x_hosts = [torch.from_numpy(host_np).pin_memory() for _ in range(args.steps)]
    for g in graphs:  # capture the host-input step graphs (record decode included) before the region
        g.capture(tuple(x_hosts[0].shape), dtype=x_hosts[0].dtype)
    outs = [[torch.empty(tuple(g._slots[0]["y"].shape), dtype=torch.float32).pin_memory()
             for _ in range(args.steps)] for g in graphs]
    for g in graphs:  # W untimed end-to-end warm-up steps (first replay of each slot's graph uploads it)
        g.run_pipelined(x_hosts[:max(2, min(args.warmup, len(x_hosts)))])
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for g, o in zip(graphs, outs):
        g.run_pipelined(x_hosts, o, before_step=flush.zero_)
    e1.record()
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    for o, t in zip(outs, ys):  # the host logits of the last e2e step == the device-timed run's
        assert torch.equal(o[-1].view(torch.int32), t.cpu().view(torch.int32))

    if args.report_out and ctx["rank"] == 0 and graphs:  # the reference harness's report (outside the region)
        from paper_2002_09481_b200.benchmark import run_benchmark
        from paper_2002_09481_b200.formats import report_csv, save_report

        report, _ = run_benchmark(graphs[0], np.concatenate([host_np] * args.steps), batch_size=batch,
                                  batches=args.steps)
        save_report(report, args.report_out + ".json")
        Path(args.report_out + ".csv").write_text(report_csv(report))

    conv_ms = sum(a.elapsed_time(b) for _, a, b, _, _, _ in profile) / args.steps
    extra = {"profile": profile, "mprofile": mprofile, "clocks": clocks, "tuned": tuned, "graphs": graphs,
             "h2d": int(x_hosts[0].numel() * x_hosts[0].element_size() * len(graphs)),
             "d2h": int(sum(o[0].numel() * 4 + g.flags.numel() * 4 for g, o in zip(graphs, outs))),
             "e2e_path": "GpuGraph.run_pipelined: pinned host batch ("
                         + ("CIFAR-10 binary records, decoded on the device" if spec["kind"] == "cifar"
                            else "fp32 NHWC images")
                         + "), H2D on a copy stream overlapping the previous step, CUDA-graph step, D2H of "
                           "logits + flags; L2 flushed before every step inside the region"}
    return {"total_ms": total_ms, "e2e_ms": e2e_ms, "conv_ms": conv_ms, "logits": y, "labels": labels,
            "launches": launches, "extra": extra}


# ---------------------------------------------------------------------------- roofline / HBM blocks


def roofline_block(args, res, sm_count, max_mhz, sampled, total_ms):
    prof = res["extra"]["profile"]
    steps = args.steps
    conv_ms = sum(a.elapsed_time(b) for _, a, b, _, _, _ in prof) / steps
    conv_macs = sum(m for _, _, _, m, _, _ in prof) / steps
    conv_algo_bytes = sum(ab for *_, ab, _ in prof) / steps
    launches = len(prof) // steps
    theo = sm_count * 64 * max_mhz * 1e6
    lds16 = sm_count * 32 * max_mhz * 1e6
    measured = {}
    try:
        measured = json.loads((ROOT / "profiles" / "smem_roofline.json").read_text())["products_per_s"]
    except Exception:
        measured = {}
    peak = max(measured.get("lds64", 0.0), measured.get("lds128", 0.0)) or theo
    achieved = conv_macs / (conv_ms / 1e3) if conv_ms else 0.0
    # per kernel family: launches, average launch, share of the step
    fam: dict = {}
    for _, a, b, m, _, k in prof:
        r = fam.setdefault(k, [0, 0.0, 0])
        r[0] += 1
        r[1] += a.elapsed_time(b)
        r[2] += m
    step_ms = total_ms / steps
    kernels = {k: {"launches_per_step": v[0] // steps, "avg_us": round(v[1] / v[0] * 1e3, 2),
                   "share_of_step": round(v[1] / steps / step_ms, 4),
                   "glookup_s": round(v[2] / (v[1] / 1e3) / 1e9, 1)} for k, v in fam.items()}
    dominant = max(kernels, key=lambda k: kernels[k]["share_of_step"]) if kernels else None
    traffic = None
    tf = ROOT / "profiles" / f"traffic_{args.workload}.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    conflict = None
    cf = ROOT / "profiles" / "conflicts.json"
    if cf.exists():
        try:
            captured = json.loads(cf.read_text()).get(args.workload, [])
            if captured:
                conflict = sum(x["bank_conflict_wavefronts"] for x in captured) / sum(
                    x["shared_ld_wavefronts"] for x in captured)
        except Exception:
            conflict = None
    return {
        "bound": "smem", "kernel": "LUT-product gather conv, all conv launches of a step",
        "dominant_kernel": dominant, "kernels": kernels,
        "achieved": round(achieved / 1e9, 2), "peak": round(peak / 1e9, 2), "unit": "Glookup/s",
        "frac": round(achieved / peak, 4),
        "frac_at_sampled_clock": round(achieved / peak * max_mhz / sampled, 4) if sampled else None,
        "peak_basis": ("measured: conflict-free LDS.64/LDS.128 warp gathers of 16-bit products "
                       "(profiles/smem_roofline.json, scripts/smem_roofline.cu)") if measured else
                      (f"derived: {sm_count} SMs x 128 B/clk / 2 B per product x {max_mhz:.0f} MHz"),
        "peak_theoretical": round(theo / 1e9, 2),
        "peak_lds32_gather_measured": round(measured["lds32"] / 1e9, 2) if measured else None,
        "lds_conflict_wavefront_frac": round(conflict, 4) if conflict is not None else None,
        "conflict_basis": "profiles/conflicts.json (ncu l1tex shared-load bank conflicts / wavefronts)",
        "lds16_lookup_roofline": round(lds16 / 1e9, 2),
        "frac_vs_lds16_lookup_roofline": round(achieved / lds16, 4),
        "traffic": traffic,
        "traffic_unit": ("DRAM bytes per LUT-conv launch: ncu dram__bytes_read.sum + dram__bytes_write.sum averaged "
                         "over one step's conv launches (cold cache, tuned kernels; profiles/traffic_<workload>.json)"),
        "algorithmic_bytes_per_launch": int(conv_algo_bytes / max(launches, 1)),
        "conv_launches_per_step": launches,
        "conv_share_of_step": round(conv_ms / step_ms, 4) if total_ms else None,
    }


def hbm_block(args, res, peak_gbs):
    """GB/s of the memory-bound kernels (range, record decode, quantize, pools, add) from the eager
    pass: algorithmic bytes (4 B per fp32 element read / written, 1 B per code) / event-timed launch;
    for the quantizer also the committed ncu launch-list durations of the same kernels (no event
    overhead; profiles/quantize_ncu_<workload>.json)."""
    agg: dict = {}
    # the depthwise conv does 9 lookups per output: it is memory-bound too (codes in, fp32 out)
    dw = [(nid, k, a, b, ab) for nid, a, b, _, ab, k in res["extra"]["profile"] if k.startswith("depthwise")]
    for _, kind, a, b, nbytes in list(res["extra"]["mprofile"]) + dw:
        r = agg.setdefault(kind, [0, 0.0, 0])
        r[0] += 1
        r[1] += a.elapsed_time(b)
        r[2] += nbytes
    out = {"peak_gbs": peak_gbs, "peak_basis": "MEASURED_PEAKS.json hbm_gbs (copy test)", "kernels": {}}
    tb = tm = 0.0
    for k, (n, ms, nb) in sorted(agg.items()):
        gbs = nb / (ms / 1e3) / 1e9 if ms else 0.0
        out["kernels"][k] = {"launches_per_step": n // args.steps, "ms_per_step": round(ms / args.steps, 4),
                             "bytes_per_step": int(nb / args.steps), "gbs": round(gbs, 1),
                             "frac": round(gbs / peak_gbs, 4) if peak_gbs else None}
        tb += nb
        tm += ms
    qf = ROOT / "profiles" / f"quantize_ncu_{args.workload}.json"  # same kernels' ncu launch-list durations
    if "quantize" in out["kernels"] and qf.exists():
        try:
            qn = json.loads(qf.read_text())
            q = out["kernels"]["quantize"]
            gbs = q["bytes_per_step"] / (qn["ms_per_step"] / 1e3) / 1e9
            q["ncu_launch_list"] = {"ms_per_step": qn["ms_per_step"], "gbs": round(gbs, 1),
                                    "frac": round(gbs / peak_gbs, 4) if peak_gbs else None,
                                    "basis": qn["source"]}
        except Exception:
            pass
    out["all"] = {"gbs": round(tb / (tm / 1e3) / 1e9, 1) if tm else None,
                  "frac": round(tb / (tm / 1e3) / 1e9 / peak_gbs, 4) if tm and peak_gbs else None,
                  "share_of_step": round(tm / res["total_ms"], 4) if res["total_ms"] else None}
    return out


def parity_block(args, spec, batch, y_rank0) -> dict:
    """Rank 0's logits vs the real reference's for the same batch (tests/golden/bench.npz)."""
    path = ROOT / "tests" / "golden" / "bench.npz"
    # goldens: <workload>_* for truncated_lut(signed, 2) (and the sweep), <workload>exact_* for exact_lut
    tag = args.workload if args.lut == "trunc2" or spec.get("sweep") else f"{args.workload}{args.lut}"
    key = f"{tag}_logits_sha"
    if batch != spec["batch"] or args.lut == "random" or not path.exists():
        return {"status": "unchecked", "why": "no reference golden for this workload / batch / table"}
    g = np.load(path)
    if key not in g:
        return {"status": "unchecked", "why": f"{key} missing from tests/golden/bench.npz"}
    got = np.ascontiguousarray(y_rank0.reshape(batch, 1, 1, -1).astype(np.float32))
    sha = hashlib.sha256(got.tobytes()).digest()
    am = got.reshape(batch, -1).argmax(1)
    ok = sha == g[key].tobytes() and np.array_equal(am, g[f"{tag}_argmax"])
    what = ("the sweep's first candidate network (truncated_lut(signed, 0))" if spec.get("sweep") else
            f"the same batch, weights and table ({spec['lut']})")
    return {"status": "bit-exact" if ok else "MISMATCH",
            "against": f"tests/golden/bench.npz {key}: sha256 of all {batch} logits rows from the real reference "
                       f"graph.run (engine gemm) on {what}",
            "logits_sha256": sha.hex(), "argmax_distinct_classes": int(len(set(am.tolist())))}


# ---------------------------------------------------------------------------- main


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="r50", choices=["r8", "r50", "r62", "r62sweep", "mbv1"])
    ap.add_argument("--lut", default="trunc2", choices=["trunc2", "exact", "random"])
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--stub", action="store_true", help="CPU/gloo synthetic step: launcher + sharding + JSON only")
    ap.add_argument("--share-device", action="store_true",
                    help="test mode: every rank on cuda:0 with gloo collectives (the multi-rank device path on a "
                         "one-GPU box; its timings are not a scaling measurement)")
    ap.add_argument("--launch", action="store_true",
                    help="re-launch under torch.distributed.run even for --gpus 1: the process group (NCCL) and "
                         "the logits/counts exchange then run with a single rank (evidence on a one-GPU box)")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-numba", action="store_true", help="skip the real-reference (numba) CPU timing")
    ap.add_argument("--layers-out", default="")
    ap.add_argument("--no-autotune", action="store_true", help="use the cost model's kernel variants")
    ap.add_argument("--tuned-out", default="", help="write the autotuned per-layer variants (json)")
    ap.add_argument("--tuned-from", default="", help="use per-layer variants from a --tuned-out file")
    ap.add_argument("--report-out", default="",
                    help="also write a RunReport (t_init + t_comp, phase split; reference bench.py:37-87) of "
                         "benchmark.run_benchmark over --steps batches: <path>.json and <path>.csv")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3

    if "WORLD_SIZE" not in os.environ and (args.gpus > 1 or args.launch):
        if args.impl == "reference":  # the CPU arm runs once, on "rank 0"
            os.environ.update(WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
        else:
            sys.exit(launch_ranks(args, argv))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if args.share_device else int(os.environ.get("LOCAL_RANK", "0"))
    spec = workload_spec(args.workload, args.lut)
    batch = args.batch or spec["batch"]
    from paper_2002_09481_b200 import resnet

    macs_img = resnet.macs_per_image(spec["nodes"])
    if args.impl == "reference":
        return reference_arm(args, spec, batch, world, rank, macs_img)

    import torch

    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    dist = None
    if args.stub:
        dev = torch.device("cpu")
    else:
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
    if world > 1 or "TORCHELASTIC_RUN_ID" in os.environ:  # launched ranks (also a one-rank --launch)
        import torch.distributed as dist

        if args.stub or args.share_device:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if dist is not None:
            dist.barrier()
        if not args.stub:
            torch.cuda.synchronize()

    ctx = {"rank": rank, "world": world, "device": dev, "barrier": barrier}
    units = units_of(spec, world, rank)
    res = (stub_rank if args.stub else device_rank)(args, spec, batch, ctx, units)

    # ------------------------------------------------ max over ranks, NCCL gather of logits/counts
    from paper_2002_09481_b200.dist import exchange_results

    logits = res["logits"] if isinstance(res["logits"], torch.Tensor) else torch.from_numpy(res["logits"])
    logits = logits.to(dev)
    labels = np.asarray(res["labels"]).astype(np.int64)
    pred = logits.argmax(-1).cpu().numpy() if logits.numel() else np.zeros((0, batch), np.int64)
    agree = (pred == labels[None, :]).sum(1) if len(pred) else np.zeros(0, np.int64)
    cnt = torch.tensor([int(agree.sum()), batch * len(units)], dtype=torch.int64, device=dev)
    t = torch.tensor([res["total_ms"], res["e2e_ms"], res["conv_ms"]], dtype=torch.float64, device=dev)
    if args.share_device:  # gloo collectives: host tensors
        logits, cnt, t = logits.cpu(), cnt.cpu(), t.cpu()
    gathered, cnt, t = exchange_results(logits, cnt, t)
    unit_lists = [units]
    if dist is not None:
        unit_lists = [None] * world
        dist.all_gather_object(unit_lists, units)
    total_ms, e2e_ms, _ = (float(v) for v in t.tolist())
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    nets_total = sum(len(u) for u in unit_lists)
    images = batch * nets_total * args.steps  # image x network evaluations over all ranks
    gmacs = images * macs_img / (total_ms / 1e3) / 1e9
    e2e_gmacs = images * macs_img / (e2e_ms / 1e3) / 1e9
    flat = sorted(i for u in unit_lists for i in u)
    units_info = {"kind": "candidate tables" if spec.get("sweep") else "range-batches",
                  "per_rank": [len(u) for u in unit_lists], "total": nets_total,
                  "covered_once": flat == list(range(32 if spec.get("sweep") else 1)) if spec.get("sweep")
                  else nets_total == world}
    line = {
        "metric": METRIC, "value": round(gmacs, 2), "unit": "GMAC/s",
        "images_per_s": round(images / (total_ms / 1e3), 2), "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        # range-batches: fixed batch per GPU (weak); the 32-table sweep: fixed job split over ranks (strong)
        "scaling": "strong" if spec.get("sweep") else "weak",
        "vs_baseline": round(gmacs / PAPER_GMACS[args.workload], 2) if args.workload in PAPER_GMACS else None,
        "vs_baseline_basis": ("paper-derived GTX 1080 approx GMAC/s (BASELINE.md s1)"
                              if args.workload in PAPER_GMACS else "no published number for this config"),
        "dtype": "u8", "data": "synthetic",
        "config": make_config(spec, args, batch, world, macs_img),
        "units": units_info,
        "agreement_with_labels": round(float(cnt[0]) / float(cnt[1]), 4) if float(cnt[1]) else None,
    }
    if dist is not None:  # the one exchange after the timed work (dist.exchange_results)
        line["exchange"] = {"backend": dist.get_backend(), "ranks": world,
                            "ops": "all_gather(unit counts, logits) + all_reduce(counts SUM, times MAX)",
                            "logits_rows_gathered": sum(int(g.shape[0]) for g in gathered)}
    if args.stub:
        line["stub"] = "synthetic host step (no GPU): launcher, sharding, gather and JSON path only"
        line["logits_gathered"] = list(gathered.shape) if hasattr(gathered, "shape") else [len(gathered)]
        print(json.dumps(line), flush=True)
        if dist is not None:
            dist.destroy_process_group()
        return

    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    ex = res["extra"]
    clocks = ex["clocks"]
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    max_mhz = float(peaks.get("sm_max_mhz") or clocks.get("sm_max_mhz") or 1965.0)
    y0 = res["logits"][0].cpu().numpy() if len(units) else None
    line["parity"] = parity_block(args, spec, batch, y0) if y0 is not None else {"status": "unchecked"}
    if args.share_device:
        line["shared_device"] = True  # test mode: all ranks on cuda:0 (not a scaling measurement)
    # rank 0's device time alone feeds the per-kernel blocks (same GPU model on every rank)
    line["roofline"] = roofline_block(args, res, sm_count, max_mhz, clocks.get("sm_mhz"), res["total_ms"])
    hbm_peak = float(peaks.get("hbm_gbs") or 6550.0)
    line["hbm"] = hbm_block(args, res, hbm_peak)
    line["config_detail"] = {"step": "one CUDA-graph replay of the whole graph (captured after warm-up)",
                             "kernel_variants": "autotuned per layer on the first batch" if ex["tuned"] else
                             "cost model"}
    line["e2e"] = {"value": round(e2e_gmacs, 2), "unit": "GMAC/s", "images_per_s": round(images / (e2e_ms / 1e3), 2),
                   "h2d_bytes_per_step": ex["h2d"], "d2h_bytes_per_step": ex["d2h"], "path": ex["e2e_path"]}
    line["gpu_launches"] = res["launches"] * args.steps
    line["clocks"] = clocks
    if world == 1 and not args.no_cpu_baseline:
        cb = cpu_reference_rate(spec, macs_img, budget_s=args.cpu_budget)
        for k in ("images", "seconds"):
            cb.pop(k, None)
        if not args.no_numba:
            nb = reference_numba_rate(spec, macs_img, budget_s=min(args.cpu_budget, 10.0))
            if nb is not None:
                cb["reference_numba"] = nb
        line["cpu_baseline"] = cb
    if args.layers_out:
        g0 = ex["graphs"][0]
        picks = g0.tuning()
        peak = line["roofline"]["peak"] * 1e9
        rows = {}
        for nid, a, b, m, _, _ in ex["profile"]:
            r = rows.setdefault(nid, [0.0, 0, 0])
            r[0] += a.elapsed_time(b)
            r[1] += m
            r[2] += 1
        Path(args.layers_out).write_text(json.dumps(
            [{"node": k, "variant": lib_variant_name(picks.get(k, 0)), "ms": round(v[0] / v[2], 4),
              "gmacs": round(v[1] / (v[0] / 1e3) / 1e9, 1), "frac": round(v[1] / (v[0] / 1e3) / peak, 4)}
             for k, v in rows.items()], indent=1))
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    if line["parity"]["status"] == "MISMATCH":
        sys.exit(3)


if __name__ == "__main__":
    main()
