#!/usr/bin/env python
"""Benchmark: certified sentences/s (full cmd_maxeps epsilon bisection per sentence) on the
BASELINE.json 3-layer workload (c3: d=256, ffn=512, seq 64, two words l1-perturbed), plus
ms per bound pass.  One "step" = the epsilon search of one batch of synthetic sentences per
GPU (each sentence 22 bound passes unless eps_max verifies).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]

Multi-GPU: one process per GPU.  Under torchrun (WORLD_SIZE set) each process is one rank;
`--gpus N` without torchrun re-launches this script under `torch.distributed.run` with N ranks.
Sentences are sharded across ranks with no data-path collective ("scaling": "weak");
torch.distributed only provides the barrier and the max-over-ranks of the device time.
Verdicts are decision-exact (fg_model_set_exact_resolve, on by default): ambiguous probes are
re-decided by the exact pass inside the timed region.  `--impl reference` times the reference's
own CPU path (oracle/_ref, the unmodified reference build) on the host cores, rank 0 only: one
complete bound pass per host thread, advanced node by node across the timed steps (measured,
not extrapolated from a prefix).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# stdout carries exactly one JSON line: NCCL's own logging goes to stderr (INFO, so the
# communicator size of a multi-GPU run is visible in the log)
os.environ.setdefault("NCCL_DEBUG", "INFO")
os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")

from paper_2209_12708_b200.configs import CONFIGS  # noqa: E402

# Our arm's bounded CPU sample: the first SAMPLE_NODES nodes of the word-level bound pass
# (layer-1 Q, K, V propagate_affine), scaled to a pass with the single-thread calibration
# profiles/cpu_calibration.json -- reported as extrapolated; the reference arm measures full passes.
SAMPLE_NODES = 3
CALIB_PATH = os.path.join(ROOT, "profiles", "cpu_calibration.json")
METRIC = "certified sentences/sec (eps binary search)"


def load_calibration(name):
    try:
        with open(CALIB_PATH) as f:
            return json.load(f)[name]
    except (OSError, KeyError, ValueError):
        return None


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def host_cpu() -> dict:
    """CPU model, logical CPUs and threads per core of this host."""
    model, tpc = "", None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Thread(s) per core:"):
                tpc = int(ln.split(":")[1])
    except (OSError, ValueError, subprocess.SubprocessError):
        pass
    return {"model": model, "logical_cpus": os.cpu_count(), "threads_per_core": tpc}


def search_passes(w) -> int:
    """Bound passes of one cmd_maxeps search (cli.cpp:159-176): verified_at(0), verified_at(eps_max),
    then one per bisection step while hi - lo > tol: 2 + ceil(log2(eps_max / tol)) whenever eps_max
    does not verify (every c2-c5 sentence; our arm reports the measured passes_per_sentence)."""
    return 2 + int(math.ceil(math.log2(w.eps_max / w.tol)))


# ---------------------------------------------------------------------------
# algorithmic work per sentence-pass
# ---------------------------------------------------------------------------
def affine_flops(w) -> float:
    """Useful flops of the bound GEMMs: 4*L*C*O*D per affine (both bounds, one product each).
    The first layer's Q/K/V affine acts on the one-hot Λ0 and is a scatter of W, not a GEMM
    (DESIGN.md §5), so it is not counted."""
    L, E, F, D = w.length, w.embed, w.ffn, w.pert_dim
    per_layer = 4.0 * L * D * (E * 3 * E + E * E + E * F + F * E)
    return w.layers * per_layer - 4.0 * L * D * E * 3 * E


def site_bytes(w) -> dict:
    """Algorithmic HBM bytes per sentence-pass of the memory-bound sites: f32 Λ, two planes,
    each Λ a site must read counted once and each Λ it produces written once.  Layer 1 is
    sparse: Λ0 is one-hot, so only the W perturbed token rows of Q/K/V carry Λ; the layer-1
    concretization reads those rows only and the layer-1 similarity product gathers only those
    Q/K rows, so those are the bytes counted there."""
    L, E, F, H, D, W = w.length, w.embed, w.ffn, w.heads, w.pert_dim, w.words
    lam = 2 * 4 * D
    deep = w.layers - 1
    return {
        "concretize": (deep * L + W) * 3 * E * lam,                                     # read Q/K/V rows
        "dot_similarity": (deep * 2 * L * E + 2 * W * E + w.layers * H * L * L) * lam,  # read Q, K; write scores
        "softmax": w.layers * 2 * H * L * L * lam,                                      # read + write scores
        "dot_weighted": w.layers * (H * L * L + 2 * L * E) * lam,                       # read P, V; write context
        "act_verify": w.layers * 2 * L * F * lam,                                       # read + write FFN Λ
    }


# ---------------------------------------------------------------------------
# clocks sampling during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active," \
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.device)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU paths (reference build / port) on the host cores
# ---------------------------------------------------------------------------
def cpu_sample(w, n_threads: int, first_sentence: int):
    """Our arm's bounded sample: the SAMPLE_NODES-node prefix of the bound pass for n_threads
    sentences concurrently (one per host thread, single-threaded each like the reference).
    Returns (wall_s, kind)."""
    import ctypes as C
    from oracle.oracle import LIBS, NORM, ModelConfig, Oracle, _d, _i
    kind = "reference" if os.path.exists(LIBS["reference"]) else "port"
    o = Oracle(kind)
    o.lib.fo_bound_pass_prefix.restype = C.c_int
    o.lib.fo_bound_pass_prefix.argtypes = None
    cfg = ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
    params = o.gen_model(cfg, w.model_seed)
    inputs = []
    for i in range(n_threads):
        s = first_sentence + i
        inputs.append((o.gen_input(cfg, w.input_seed(s)),
                       np.ascontiguousarray(o.gen_positions(w.position_seed(s), w.length, w.words), dtype=np.int32)))
    fc = cfg.fo()

    def run(i):
        x, pos = inputs[i]
        o.lib.fo_bound_pass_prefix(C.byref(fc), _d(params), _d(x), _i(pos), w.words, NORM[w.norm],
                                   C.c_double(w.eps), SAMPLE_NODES)

    threads = [threading.Thread(target=run, args=(i,)) for i in range(n_threads)]
    t0 = time.perf_counter()
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    return time.perf_counter() - t0, kind


# configs whose complete reference pass fits the bench (c3: ~90 s on 16 host threads); c4 / c5 passes
# take hours on a host core, so their baseline stays an extrapolated prefix sample
FULL_PASS_BASELINE = ("c1", "c2", "c3")


def sustained_mma_peak(ctx, local_rank: int, seconds: float = 3.0):
    """Dense kind::tf32 tcgen05 throughput under sustained load: fg_selftest_mma_peak back to back
    for `seconds`, median of the second half of the runs (the part settles at its power-capped
    clock), with the median SM clock sampled meanwhile."""
    runs = []
    with ClockSampler(local_rank) as clk:
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < seconds:
            runs.append(ctx.mma_peak("tf32", iters=100_000)["tflops"])
    half = runs[len(runs) // 2:] or runs
    return statistics.median(half), clk.summary().get("sm_mhz")


def pass_over_sample(w, kind):
    cal = load_calibration(w.name) or {}
    return (cal.get(kind) or cal.get("reference") or cal.get("port") or {}).get("pass_over_sample")


def paced_full_pass(w, n_threads: int, first_sentence: int, steps: int, warmup: int):
    """One COMPLETE word-level bound pass of the unmodified reference per host thread, all
    running concurrently; the walks advance a slice of nodes per timed step (fo_paced_step), so
    the timed steps together cover exactly one full pass per thread.  Returns per-step walls."""
    import ctypes as C
    from oracle.oracle import NORM, ModelConfig, Oracle
    o = Oracle("reference")
    L = o.lib
    L.fo_paced_begin.restype = C.c_void_p
    L.fo_paced_begin.argtypes = [C.c_void_p] * 4 + [C.c_int, C.c_int, C.c_double]
    L.fo_paced_step.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_int]
    L.fo_paced_end.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    cfg = ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
    params = o.gen_model(cfg, w.model_seed)
    fc = cfg.fo()
    keep = []

    def begin(first, n):
        hs = []
        for i in range(n):
            s = first + i
            x = o.gen_input(cfg, w.input_seed(s))
            pos = np.ascontiguousarray(o.gen_positions(w.position_seed(s), w.length, w.words), dtype=np.int32)
            keep.append((x, pos))
            hs.append(L.fo_paced_begin(C.byref(fc), params.ctypes.data, x.ctypes.data, pos.ctypes.data, w.words,
                                       NORM[w.norm], w.eps))
        return hs, (C.c_void_p * n)(*hs)

    nodes = w.layers * 16 + 2  # nodes of the walk (fo_bound_pass node order)
    # warm-up steps: the first node of a separate set of walks (pages in the library / weights)
    whs, warr = begin(first_sentence + 10_000, n_threads)
    for k in range(warmup):
        L.fo_paced_step(warr, n_threads, 1 if k == 0 else 0)
    for h in whs:
        L.fo_paced_end(h, 0, None, None)  # stop the warm-up walks at their next node
    hs, arr = begin(first_sentence, n_threads)
    walls = []
    for k in range(steps):
        n_k = (k + 1) * nodes // steps - k * nodes // steps
        t0 = time.perf_counter()
        L.fo_paced_step(arr, n_threads, n_k)
        walls.append(time.perf_counter() - t0)
    status = [L.fo_paced_end(h, 1, None, None) for h in hs]
    return walls, nodes, status


def reference_arm(args, w):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle.oracle import LIBS
    n_threads = os.cpu_count() or 1
    passes = search_passes(w)
    cpu = host_cpu()
    t0 = time.perf_counter()
    if os.path.exists(LIBS["reference"]):
        walls, nodes, status = paced_full_pass(w, n_threads, 20_000, args.steps, args.warmup)
        kind = "reference"
        t_pass = sum(walls)
        value = n_threads / (t_pass * passes)
        sample = (f"one complete {w.name} word-level bound pass (all {nodes} nodes, eps {w.eps:g}) per host thread, "
                  f"{n_threads} sentences concurrently on the unmodified reference build, advanced in "
                  f"{args.steps} node slices (one per timed step): full pass measured, {t_pass:.1f} s wall; "
                  f"x {passes} passes per sentence (2 + ceil(log2(eps_max/tol)), cli.cpp:159-176); "
                  f"pass statuses {sorted(set(status))}")
    else:
        walls = []
        kind = "port"
        for i in range(args.steps):
            walls.append(cpu_sample(w, n_threads, 20_000 + i * n_threads)[0])
        ratio = pass_over_sample(w, kind)
        t_pass = statistics.mean(walls) * ratio if ratio else None
        value = n_threads / (t_pass * passes) if t_pass else None
        sample = (f"EXTRAPOLATED (reference build absent): first {SAMPLE_NODES} nodes on the C restatement, "
                  f"x {ratio} (profiles/cpu_calibration.json) x {passes} passes")
    total = time.perf_counter() - t0
    line = {"impl": "reference", "metric": METRIC, "value": value,
            "unit": "sentences/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total / max(1, args.steps), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": {"workload": w.name, **w.as_dict()},
            "ms_per_bound_pass": None if t_pass is None else 1e3 * t_pass,
            "cpu_baseline": {"value": value, "unit": "sentences/s", "cores": n_threads, "kind": kind,
                             "sample": sample, "cpu": cpu},
            "e2e": {"value": value, "unit": "sentences/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# launching N ranks without torchrun
# ---------------------------------------------------------------------------
def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args) -> int:
    """`--gpus N` outside torchrun: run this script under torch.distributed.run with N ranks
    (127.0.0.1 rendezvous); rank 0's JSON line is the only stdout."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def dry_run(args, w) -> int:
    """--dry-run: the multi-rank plumbing without a GPU (gloo): rank/world, the sentence blocks and
    the max-over-ranks reduction; prints the JSON line's shape keys."""
    from paper_2209_12708_b200 import dist as D
    rank, world, _ = dist_env()
    dist = D.init(backend="gloo")
    assert world == args.gpus, f"world size {world} != --gpus {args.gpus}"
    B = args.batch or {"c1": 256, "c2": 256, "c3": 64, "c4": 16, "c5": 4}[w.name]
    ids = [list(D.sentence_block(rank, s, args.steps + args.warmup, B)) for s in range(args.steps + args.warmup)]
    first = D.max_over_ranks([ids[0][0]], dist)[0]
    line = {"metric": METRIC, "value": None, "n_gpus": world, "dry_run": True,
            "config": {"workload": w.name, "global_batch": B * world, "sentences_per_step_per_gpu": B,
                       "parallelism": f"sentence-sharded dp{world}"},
            "max_first_sentence_over_ranks": first}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=0, help="sentences per step per GPU (default: per config)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--raw-f32-verdicts", action="store_true",
                    help="decide every probe on the f32-Λ pass alone (kappa 0; comparison only: near ε* the "
                         "bisection may leave the reference's path)")
    ap.add_argument("--dry-run", action="store_true", help="multi-rank plumbing only (gloo, no GPU work)")
    ap.add_argument("--shard", default="sentences", choices=["sentences", "columns"],
                    help="sentences: independent sentences per GPU (weak scaling, no collective); columns: "
                         "perturbation columns of every sentence split over the GPUs, concretization partials "
                         "all-reduced with NCCL inside the pass (strong scaling; SURVEY 8(e) c5)")
    ap.add_argument("--speculative", type=int, default=0, metavar="DEPTH",
                    help="speculative eps bisection: DEPTH levels per batched round, the probes of a round "
                         "split over the GPUs (latency mode for few sentences, e.g. c1; SURVEY 8(e))")
    args = ap.parse_args()
    w = CONFIGS[args.config]
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch(args)
    if args.dry_run:
        return dry_run(args, w)
    if args.impl == "reference":
        return reference_arm(args, w)

    import torch
    from paper_2209_12708_b200 import dist as D
    from paper_2209_12708_b200 import faith_gpu as F

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE {world} != --gpus {args.gpus}")
    torch.cuda.set_device(local)
    dist = D.init(backend="nccl", device_index=local)
    B = args.batch or {"c1": 256, "c2": 256, "c3": 64, "c4": 16, "c5": 4}[w.name]

    cfg = F.ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
    ctx = F.Context(local)
    model = F.Model(ctx, cfg, F.gen_synthetic(cfg, w.model_seed))
    if args.raw_f32_verdicts:
        model.set_exact_resolve(0.0)
    columns = args.shard == "columns"
    spec = args.speculative > 0
    if columns:
        D.shard_model_columns(model, dist)

    def batch(step):
        # globally unique sentence ids: rank-major blocks, warm-up steps first (no data-path collective);
        # column sharding: every rank works on the same sentences (its own slice of their columns)
        ids = D.sentence_block(0 if (columns or spec) else rank, step, args.steps + args.warmup, B)
        xs = np.stack([F.gen_input(cfg, w.input_seed(i)) for i in ids])
        ps = np.stack([F.gen_positions(w.position_seed(i), w.length, w.words) for i in ids])
        return xs, ps

    inputs = [batch(s) for s in range(args.warmup + args.steps)]  # host buffers (the user's data)
    # dense TF32 tensor peak of this device, burst (before the timed region heats the part up)
    tf32_peak = max(ctx.mma_peak("tf32")["tflops"] for _ in range(3)) if rank == 0 else None

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    def search(xs, ps):
        if spec:
            return model.maxeps_speculative(xs, ps, w.norm, w.eps_max, w.tol, depth=args.speculative, dist=dist)
        return model.maxeps(xs, ps, w.norm, w.eps_max, w.tol, slots=B)

    for s in range(args.warmup):
        search(*inputs[s])
    barrier()
    dev_ms, calls, launches, passes, pass_ms, exact_probes, exact_ms = 0.0, [], 0, 0, [], 0, 0.0
    rollbacks = 0
    h2d = d2h = 0
    # fg_maxeps runs the eps = 0 probes up front on a narrow workspace (one pass for B <= 256
    # sentences) when words*embed > 128 and the pass is not column-sharded: its eps/slot staging
    # and verdict readback
    zero_probe = w.words * w.embed > 128 and not (columns or spec) and os.environ.get("FG_NO_ZERO_PROBE") != "1"
    with ClockSampler(local) as clocks:
        barrier()
        t0 = time.perf_counter()
        for s in range(args.warmup, args.warmup + args.steps):
            r = search(*inputs[s])
            st = model.last_stats()
            dev_ms += st["device_ms"]
            launches += st["launches"]
            passes += st["passes"]
            pass_ms.append(st["pass_ms"])
            exact_probes += st["exact_probes"]
            exact_ms += st["exact_ms"]
            rollbacks += st["spec_rollbacks"]
            calls.extend(r["calls"].tolist())
            # every step copies its batch's inputs in (x f64, positions i32) and the results out
            # (eps f64, calls / predicted / status i32), plus per pass the eps/slot staging and
            # the logits-bound/status readback; an exact re-decision copies one sentence in and
            # its logits out
            h2d += B * (w.length * w.embed * 8 + w.words * 4)
            d2h += B * (8 + 4 + 4 + 4)
            zp = -(-B // 256) if zero_probe else 0
            h2d += (st["passes"] + zp) * B * (8 + 4) + st["exact_probes"] * (w.length * w.embed * 8 + w.words * 4)
            d2h += (st["passes"] + zp) * B * (2 * w.classes * 8 + 4) + st["exact_probes"] * 2 * w.classes * 8
        barrier()
        wall = time.perf_counter() - t0
    dev_ms_max, wall_max = D.max_over_ranks([dev_ms, wall], dist, device="cuda")
    sentences = B * args.steps * (1 if (columns or spec) else world)
    value = sentences / (dev_ms_max / 1e3)
    e2e = sentences / wall_max
    ms_pass_batched = statistics.mean(pass_ms)
    ms_pass_sentence = ms_pass_batched / B

    line = {
        "metric": METRIC, "value": value, "unit": "sentences/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms_max / args.steps,
        "higher_is_better": True, "scaling": "strong" if (columns or spec) else "weak", "vs_baseline": None,
        "dtype": "f32+f64",
        "data": f"synthetic: gen_synthetic(seed {w.model_seed}) weights, gen_synthetic_input(2000+s), "
                f"{w.words} perturbed word(s) at Rng(3000+s) positions",
        "config": {**w.as_dict(), "global_batch": B * (1 if (columns or spec) else world),
                   "sentences_per_step_per_gpu": B,
                   "parallelism": (f"column-sharded cp{world} (NCCL all-reduce of concretization partials)"
                                   if columns else
                                   f"speculative bisection depth {args.speculative} over {world} GPU(s)" if spec
                                   else f"sentence-sharded dp{world}"),
                   "verdicts": "raw f32 (kappa 0)" if args.raw_f32_verdicts else
                               f"decision-exact (kappa {F.DEFAULT_KAPPA:g}: ambiguous probes re-decided by the "
                               "exact pass)",
                   "l2_flush": "not needed: inputs larger than L2 (Λ working set "
                               f"{B * 0.45:.1f} GB per GPU >> 126 MB L2)"},
        "ms_per_bound_pass": {"batched_pass_ms": ms_pass_batched, "per_sentence_ms": ms_pass_sentence,
                              "batch": B},
        "passes_per_sentence": statistics.mean(calls),
        "exact_probes_per_sentence": exact_probes / (B * args.steps),
        "exact_ms_share": exact_ms / dev_ms if dev_ms else 0.0,
        "speculation": {"rollbacks_per_step": rollbacks / args.steps, "batched_passes_per_step": passes / args.steps,
                        "_note": "sentences bisect on with a guessed verdict while their ambiguous probe is "
                                 "re-decided; a wrong guess rolls the sentence back (include/faith_gpu.h "
                                 "fg_model_set_speculation)"},
        "ambiguity_band": {"lo": st["band_lo"], "hi": st["band_hi"], "calibration_samples": st["band_samples"],
                           "unit": "fraction of the two logits bounds' widths"},
        "e2e": {"value": e2e, "unit": "sentences/s", "h2d_bytes_per_step": h2d // args.steps,
                "d2h_bytes_per_step": d2h // args.steps},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    if w.name in ("c4", "c5"):
        # random-init weights at these depths widen the bounds ~10^3x per layer (DESIGN.md §9,
        # profiles/r1_width_growth_by_depth.txt): the certified radius is ~0 and most probes above
        # it end in a domain error, so sentences/s here times searches of mostly failing probes
        line["workload_note"] = ("degenerate on random-init weights: certified eps ~0, probes above it mostly end "
                                 "in domain errors (early exit)")

    prof = None
    prof_clk = None
    if not args.no_profile and (rank == 0 or columns):  # column shards all-reduce inside the pass
        # five eager profiled passes (median per site) with the SM clock sampled meanwhile
        with ClockSampler(local) as pclk:
            runs = [model.profile_pass(w.norm, w.eps) for _ in range(5)]
        prof = {k: (statistics.median(r[k][0] for r in runs), runs[0][k][1]) for k in runs[0]}
        prof_clk = pclk.summary().get("sm_mhz")
    if rank == 0 and prof is not None:
        pk, pk_kind = peaks()
        tf32 = tf32_peak
        tf32_sus, tf32_clk = sustained_mma_peak(ctx, local)
        total = sum(ms for ms, _ in prof.values())
        gemm_ms, gemm_k = prof.get("affine_gemm", (0.0, 0))
        flops = affine_flops(w) * B / (world if columns else 1)
        ach = flops / (gemm_ms / 1e3) / 1e12 if gemm_ms else None
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                traffic = json.load(f).get(w.name, {}).get("affine_gemm_bytes_per_launch")
        except (OSError, ValueError):
            pass
        # the GEMM is timed inside a long step (a profiled pass right after the timed region, the
        # part power-capped): the sustained peaks are its denominators
        bf16_sus = pk.get("bf16_tflops_sustained") or pk["bf16_tflops"]
        line["roofline"] = {
            "kernel": "affine bound GEMM (propagate_affine, c/r form)", "bound": "tensor",
            "achieved": ach, "peak": bf16_sus, "unit": "TFLOP/s",
            "frac": (ach / bf16_sus) if ach else None, "traffic": traffic,
            "peak_source": f"{pk_kind} dense bf16, sustained (MEASURED_PEAKS.json; the kernel is timed inside a "
                           "long step)",
            "peak_burst": pk["bf16_tflops"], "frac_burst": (ach / pk["bf16_tflops"]) if ach else None,
            "algorithmic": f"{affine_flops(w):.4g} useful flop per sentence-pass (4*L*C*O*D per GEMM affine; "
                           f"layer-1 Q/K/V is a one-hot scatter) x {B} sentences per launch set",
            "launches_per_pass": gemm_k, "share_of_pass": gemm_ms / total if total else None,
            # the precision north_star asks for (error-compensated 3xTF32): each useful product costs
            # three kind::tf32 MMAs, so its ceiling is the measured dense TF32 rate / 3
            "peak_tf32_measured": tf32,
            "peak_tf32_source": "fg_selftest_mma_peak: tcgen05.mma kind::tf32 M128 N256, one CTA per SM, "
                                "SMEM-resident operands; burst = best of 3 before the timed region, sustained = "
                                "median of the second half of ~3 s of back-to-back runs after the profiled pass "
                                "(the same harness gives kind::f16 bf16 = 2.00 x tf32)",
            "peak_tf32_sustained": tf32_sus, "sm_mhz_during_tf32_sustained": tf32_clk,
            "peak_3xtf32": tf32_sus / 3.0,
            "frac_3xtf32": (ach / (tf32_sus / 3.0)) if ach else None,
            "peak_3xtf32_burst": tf32 / 3.0,
            "frac_3xtf32_burst": (ach / (tf32 / 3.0)) if ach else None,
            # the tcgen05 rate per clock is fixed: the ceiling at the SM clock the power cap allows
            # while the pass runs (the MMA microbenchmark alone stays at the maximum clock)
            "sm_mhz_during_profiled_pass": prof_clk,
            "frac_3xtf32_at_pass_clock": (ach / (tf32_sus / 3.0 * prof_clk / tf32_clk))
            if (ach and prof_clk and tf32_clk) else None,
        }
        mem = {}
        for site, nbytes in site_bytes(w).items():
            if site in prof and prof[site][0] > 0:
                gbs = nbytes * B / (world if columns else 1) / (prof[site][0] / 1e3) / 1e9
                mem[site] = {"GB/s": gbs, "frac_hbm": gbs / pk["hbm_gbs"], "ms": prof[site][0],
                             "algorithmic_GB": nbytes * B / 1e9}
        line["kernels"] = {k: {"ms_per_pass": v[0], "launches": v[1]} for k, v in sorted(prof.items())}
        mem["_note"] = ("GB/s = algorithmic bytes (each Λ a site reads counted once, each Λ it writes once; "
                        "layer-1 Q/K/V rows only where Λ is non-zero) / site time of one eager profiled pass; "
                        "DRAM bytes per launch are in the committed ncu launch list (profiles/)")
        line["hbm_sites"] = mem

    if rank == 0 and world == 1 and not args.no_cpu_baseline and w.name in FULL_PASS_BASELINE:
        # one complete pass per host thread of the unmodified reference build (c3: ~90 s)
        from oracle.oracle import LIBS
        n_threads = os.cpu_count() or 1
        if os.path.exists(LIBS["reference"]):
            walls, nodes, status = paced_full_pass(w, n_threads, 900_000, 1, 1)
            t_pass = sum(walls)
            rate = n_threads / (t_pass * statistics.mean(calls))
            line["cpu_baseline"] = {
                "value": rate, "unit": "sentences/s", "cores": n_threads, "kind": "reference", "cpu": host_cpu(),
                "sample": f"one complete {w.name} word-level bound pass (all {nodes} nodes, eps {w.eps:g}) per host "
                          f"thread, {n_threads} sentences concurrently on the unmodified reference build: full pass "
                          f"measured, {t_pass:.1f} s wall; x {statistics.mean(calls):.1f} passes/sentence (this "
                          f"run's mean calls); pass statuses {sorted(set(status))}"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline and "cpu_baseline" not in line:
        n_threads = os.cpu_count() or 1
        wall_cpu, kind = cpu_sample(w, n_threads, 900_000)
        ratio = pass_over_sample(w, kind)
        t_pass = wall_cpu * ratio if ratio else None
        rate = n_threads / (t_pass * statistics.mean(calls)) if t_pass else None
        cal = load_calibration(w.name) or {}
        line["cpu_baseline"] = {
            "value": rate, "unit": "sentences/s", "cores": n_threads, "kind": kind, "cpu": host_cpu(),
            "sample": f"EXTRAPOLATED: first {SAMPLE_NODES} nodes of the {w.name} bound pass for {n_threads} sentences "
                      f"concurrently ({wall_cpu:.1f} s wall) x {ratio} (full pass / sample, single-thread, "
                      f"{cal.get('host', 'build container')}: profiles/cpu_calibration.json) x "
                      f"{statistics.mean(calls):.1f} passes/sentence; bench.py --impl reference measures full passes",
        }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
