#!/usr/bin/env python
"""Benchmark of the pruned RNN-T loss hot path (fwd+bwd) on B200 — BASELINE.json metric.

One "step" = the whole hot path over one batch: rnnt_simple_loss (with am/lm grads),
rnnt_get_ranges, rnnt_prune, rnnt_pruned_loss (all grads), the batch loss combination
(rnnt_loss_sums) and, when world_size > 1, the exchange of d_w, d_b and the loss sums (NCCL
all_reduce, or NVLS multimem adds with --exchange multimem).  Workload at every N: BASELINE
configs[4] (c5) = the configs[1] (c2, LibriSpeech-shaped BPE) recipe, 32 utterances per GPU,
seeded by rank, so the 1->8 curve is one workload.  Synthetic seeded inputs (synth/).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "pruned RNN-T loss fwd+bwd frames(N·T)/sec and peak GB, 1/2/4/8 B200"
UNIT = "frames/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=0, help="override BASELINE config (1-5)")
    ap.add_argument("--profile-kernel", default="auto")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches only (no CUDA graph replay)")
    ap.add_argument("--no-priority", action="store_true", help="run the step on the default-priority stream")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "multimem"],
                    help="N > 1: how d_w / d_b / loss sums are summed over ranks (include/rnnt.h exchange modes)")
    ap.add_argument("--no-standalone", action="store_true", help="skip the serial (standalone) per-kernel times")
    ap.add_argument("--copy-streams", type=int, default=2,
                    help="e2e: H2D copy streams (the packed input tensors dealt across them: two DMA engines)")
    ap.add_argument("--workload", default="fixed", choices=["fixed", "dynamic", "full"],
                    help="dynamic: the Table-2 protocol (sorted utterances, <= 10k input frames per batch); "
                         "full: the unpruned loss with the same joiner on the c2 batch (SURVEY 8(f) f4)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload(args, world, rank):
    cfg = args.config or 5
    b = synth.make_batch(cfg, rank=rank)
    name = {2: "c2 LibriSpeech-shaped BPE (BASELINE configs[1])",
            5: "c5 data-parallel (BASELINE configs[4]): the c2 LibriSpeech-shaped BPE recipe (configs[1]), "
               "32 utterances per GPU, seeded by rank"}.get(cfg, synth.CONFIGS[cfg]["name"])
    return cfg, b, name


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) < 8:
                continue
            for nm, v in zip(names, r[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        loaded = [s for s in sm if s > 0.5 * (max(sm) if sm else 1)]
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ roofline table
def algorithmic(kernel, b):
    """Algorithmic work of one launch of ``kernel`` on batch ``b``:
    (flops, bytes).  Bytes count each input read once and each output written once (real rows /
    cells only), flops the dense contractions at their real sizes."""
    T = b.T_n.astype(np.int64)
    U1 = b.U_n.astype(np.int64) + 1
    rows = int((T * b.S).sum())                 # real band rows sum_n T_n * S
    cells = int((T * U1).sum())                 # real lattice cells
    frames, toks = int(T.sum()), int(U1.sum())
    V, J, S = b.V, b.J, b.S
    if kernel == "joiner_fwd_gemm":             # h, W in; P~ (bf16), per-row scalars out
        return 2.0 * rows * J * V, rows * J * 2 + V * J * 2 + rows * V * 2 + rows * 16
    if kernel == "joiner_dh_gemm":              # P~, h, W, row scalars in; dpre rows (fp16) out
        return 2.0 * rows * J * V, rows * V * 2 + rows * J * 2 + V * J * 2 + rows * 16 + rows * J * 2
    if kernel == "joiner_dw_gemm":              # P~, h, row scalars in; dW split partials out (one V x J)
        return 2.0 * rows * J * V, rows * V * 2 + rows * J * 2 + rows * 16 + V * J * 4
    if kernel == "simple_norm_gemm":            # E_am, E_lm (bf16 hi+lo) in; arcs + 1/S out (skewed)
        return 2.0 * cells * V * 3, (frames + toks) * V * 4 + cells * 12
    if kernel == "prune_gather":                # enc, dec rows in; h (bf16) out
        return 0.0, frames * J * 4 + toks * J * 4 + rows * J * 2
    if kernel == "simple_prep":                 # am, lm in; E hi+lo out
        return 0.0, (frames + toks) * V * 4 * 2
    if kernel == "lattice_combine":             # alpha, beta, arcs, 1/S in; px/py grads, G~, y' out
        return 0.0, cells * (4 + 4 + 8 + 4) + cells * (8 + 8)
    if kernel == "simple_am_grad_gemm":         # G~, y' (hi+lo), E_lm (hi+lo), am in; am_grad out (bf16x3 issue)
        return 2.0 * cells * V * 3, cells * 8 + toks * V * 4 + frames * V * 4 + frames * V * 4
    if kernel == "simple_lm_grad_gemm":         # G~ (hi+lo), E_am (hi+lo), lm in; lm_grad out (bf16x3 issue)
        return 2.0 * cells * V * 3, cells * 4 + frames * V * 4 + toks * V * 4 + toks * V * 4
    if kernel == "joiner_band_chunk":           # dpre rows (fp16) in (each once); d_enc rows and the d_dec partials out
        return 0.0, rows * J * 2 + frames * J * 4
    if kernel == "joiner_band_dec":             # d_dec rows out (the partials read are the chunking's cost)
        return 0.0, toks * J * 4
    if kernel == "joiner_dw_reduce":            # d_w out (the split-K partials it reads are the split's cost)
        return 0.0, V * J * 4
    raise KeyError(kernel)


PROFILED = ["joiner_dh_gemm", "joiner_fwd_gemm", "joiner_dw_gemm", "simple_norm_gemm", "simple_am_grad_gemm",
            "simple_lm_grad_gemm", "prune_gather", "lattice_combine", "simple_prep", "joiner_band_chunk", "joiner_band_dec",
            "joiner_dw_reduce", "lattice_fb", "pruned_fb"]
LATENCY_BOUND = {"lattice_fb", "pruned_fb"}   # dependent log-add chains


def roofline(kernel, b, ms, hbm, tfl):
    """Roofline of one kernel from its live mean launch time: the binding resource is the one whose
    floor (algorithmic work / measured peak) is larger."""
    flops, byts = algorithmic(kernel, b)
    ft = flops / (tfl * 1e12) if flops else 0.0
    fh = byts / (hbm * 1e9)
    s = ms / 1000.0
    if ft >= fh:
        return {"kernel": kernel, "bound": "tensor", "achieved": flops / s / 1e12, "peak": tfl, "unit": "TFLOP/s",
                "frac": ft / s, "kernel_ms": ms, "algorithmic_flops": flops, "algorithmic_bytes": byts}
    return {"kernel": kernel, "bound": "hbm", "achieved": byts / s / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": fh / s, "kernel_ms": ms, "algorithmic_flops": flops, "algorithmic_bytes": byts}


def ncu_traffic(kernel, cfg):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of ``kernel`` from the
    committed ncu --set full capture summary (profiles/ncu_traffic.json), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None, None
    d = json.load(open(path))
    e = d.get(f"c{cfg}", {}).get(kernel)
    return (e["bytes"], e["source"]) if e else (None, None)


def peaks():
    """HBM copy bandwidth and the BURST bf16 dense peak (the kernels are timed inside a sub-ms step,
    not back to back for seconds), from MEASURED_PEAKS.json, else the profiling guide's fallbacks."""
    p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    return (p.get("hbm_gbs", 6650.0), p.get("bf16_tflops", 1650.0),
            "MEASURED_PEAKS.json hbm_gbs / bf16_tflops (burst)" if p else "B200_PROFILING.md fallback")


# ------------------------------------------------------------------ CPU oracle timing
_ORACLE_BATCH = None


def _oracle_init(cfg, rank):
    """Pool worker: BLAS limited to one thread (the pool supplies the parallelism), the batch drawn
    from its seed (nothing large crosses the process boundary)."""
    global _ORACLE_BATCH
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(limits=1)
    except Exception:
        pass
    import oracle  # noqa: F401  (import cost outside the timed region)
    _ORACLE_BATCH = synth.make_batch(cfg, rank=rank)


def _oracle_utt(n):
    """The whole oracle path for utterance n (as it stands): simple loss + grads, Eq. 8, ADJ-scan,
    pruned loss + grads.  Returns its frame count."""
    import oracle as O
    d = _ORACLE_BATCH.utterance(n)
    s = O.simple_loss(d["am"], d["lm"], d["y"], 0.5)
    pxg, pyg = s["px_grad"].astype(np.float32), s["py_grad"].astype(np.float32)
    if O.feasible(d["T"], d["U"], d["S"]):
        p = O.adjust_bounds(O.raw_bounds(pxg, pyg, d["S"]), d["T"], d["U"], d["S"])
        O.pruned_loss(d["enc"], d["dec"], d["W"], d["b"], d["y"], p, d["S"], 1.0, matched=True)
    return d["T"]


def _noop(_):
    return 0


class OraclePool:
    """The fp64 oracle on every host core: a process pool over utterances."""

    def __init__(self, cfg, rank=0):
        import concurrent.futures as cf
        import multiprocessing as mp
        self.cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
        self.ex = cf.ProcessPoolExecutor(self.cores, mp_context=mp.get_context("spawn"),
                                         initializer=_oracle_init, initargs=(cfg, rank))
        list(self.ex.map(_noop, range(4 * self.cores)))          # workers up, batch drawn
        self.next = 0

    def run(self, seconds, N, max_utts=None):
        """Utterances (rotating over the batch) with ``cores`` in flight until ``seconds`` of wall time
        (or ``max_utts``); returns (frames/s, frames, utterances, elapsed)."""
        import concurrent.futures as cf
        t0 = time.perf_counter()
        frames, done, pending = 0, 0, set()
        submitted = 0
        while True:
            stop = time.perf_counter() - t0 >= seconds or (max_utts is not None and submitted >= max_utts)
            while not stop and len(pending) < self.cores:
                pending.add(self.ex.submit(_oracle_utt, self.next % N))
                self.next += 1
                submitted += 1
                stop = max_utts is not None and submitted >= max_utts
            if not pending:
                break
            fin, pending = cf.wait(pending, return_when=cf.FIRST_COMPLETED)
            for f in fin:
                frames += f.result()
                done += 1
        el = time.perf_counter() - t0
        return frames / el, frames, done, el

    def close(self):
        self.ex.shutdown()


# ------------------------------------------------------------------ reference arm
def run_reference(args, world, rank):
    if rank != 0:
        return 0
    cfg, b, name = workload(args, 1, 0)
    steps, warm = args.steps, args.warmup
    pool = OraclePool(cfg, 0)
    per_step = pool.cores  # utterances per step: one per host core, a bounded sample of the batch
    for _ in range(warm):
        pool.run(1e9, b.N, max_utts=per_step)
    frames = 0
    t0 = time.perf_counter()
    for _ in range(steps):
        _, f, _, _ = pool.run(1e9, b.N, max_utts=per_step)
        frames += f
    el = time.perf_counter() - t0
    pool.close()
    v = frames / el
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": steps, "warmup": warm, "ms_per_step": 1000 * el / steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": name, "N": b.N, "V": b.V, "J": b.J, "S": b.S,
                       "sample": f"{per_step} utterance(s) of the batch per step (one per host core), rotating"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": pool.cores, "kind": "oracle",
                             "sample": f"{steps} steps x {per_step} utterances, fp64 numpy, a process pool over "
                                       f"utterances on {pool.cores} cores, BLAS 1 thread per process"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ dynamic-batch workload
def run_dynamic(args):
    """Every batch of the synthetic dynamic-batch corpus (synth.make_dynamic_corpus)
    through the whole hot path, one batch per step; frames/s over the corpus and mean ms per batch."""
    import torch
    import paper_2206_13236_b200 as R
    corpus = synth.make_dynamic_corpus()
    devs = [R.batch_to_device(b, "cuda") for b in corpus]
    dims = [R.make_dims(b.N, b.T, b.U, b.V, b.J, b.S) for b in corpus]
    outs = [R.alloc_outputs(d, "cuda") for d in dims]
    ws = torch.empty(max(R.rnnt_workspace_bytes(d) for d in dims), dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step(i):
        b, dv, o = corpus[i], devs[i], outs[i]
        o["status"].zero_()
        R.step(dv["am"], dv["lm"], dv["symbols"], dv["boundary"], dv["enc_proj"], dv["dec_proj"], dv["w_out"],
               dv["b_out"], b.S, out=o, workspace=ws)

    for i in range(max(args.warmup, 3)):
        step(i % len(corpus))
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in corpus]
    clocks = Clocks(0)
    clocks.start()
    time.sleep(0.3)
    for i in range(len(corpus)):
        flush.zero_()
        ev[i][0].record()
        step(i)
        ev[i][1].record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = [a.elapsed_time(c) for a, c in ev]
    frames = sum(int(b.T_n.sum()) for b in corpus)
    peak = torch.cuda.max_memory_allocated() / 2 ** 30 - flush.numel() / 2 ** 30
    line = {"metric": METRIC, "value": frames / (sum(ms) / 1000.0), "unit": UNIT, "n_gpus": 1, "steps": len(corpus),
            "warmup": max(args.warmup, 3), "ms_per_step": statistics.mean(ms), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16+f32", "data": "synthetic",
            "config": {"workload": "dynamic batches (Table 2 protocol): c2-shaped utterances sorted by length, "
                                   f"<= {synth.DYNAMIC_CAP_FRAMES} encoder frames (10k input frames) per batch",
                       "batches": len(corpus), "utterances": sum(b.N for b in corpus), "frames": frames,
                       "padded_frames": sum(b.N * b.T for b in corpus), "V": 500, "J": 512, "S": 5,
                       "l2": "flushed between timed batches (256 MiB write, outside the timed events)",
                       "kernels": R.rnnt_version()},
            "peak_gib": peak, "clocks": clk,
            "ms_per_batch": {"mean": statistics.mean(ms), "min": min(ms), "max": max(ms)}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ full (unpruned) loss
def run_full(args):
    """The full RNN-T loss (every (t,u) through the joiner) on the c2 batch: the
    in-house counterpart of the paper's unpruned baselines (Tables 1-2), same metric and timing rules."""
    import torch
    import paper_2206_13236_b200 as R
    b = synth.make_batch(2)
    dev = R.batch_to_device(b, "cuda")
    dims = R.make_dims(b.N, b.T, b.U, b.V, b.J, 1)
    f32 = dict(dtype=torch.float32, device="cuda")
    o = dict(loss=torch.empty(b.N, **f32), d_enc=torch.empty(b.N, b.T, b.J, **f32),
             d_dec=torch.empty(b.N, b.U + 1, b.J, **f32), d_w=torch.empty(b.V, b.J, **f32),
             d_b=torch.empty(b.V, **f32), status=torch.zeros(b.N, dtype=torch.int32, device="cuda"))
    ws = torch.empty(R.rnnt_full_workspace_bytes(dims), dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step():
        R.rnnt_full_loss(dev["enc_proj"], dev["dec_proj"], dev["w_out"], dev["b_out"], dev["symbols"],
                         dev["boundary"], dims, 1.0, o["loss"], o["d_enc"], o["d_dec"], o["d_w"], o["d_b"],
                         o["status"], ws)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    clocks = Clocks(0)
    clocks.start()
    time.sleep(0.3)
    for i in range(K):
        flush.zero_()
        ev[i][0].record()
        step()
        ev[i][1].record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = [a.elapsed_time(c) for a, c in ev]
    frames = int(b.T_n.sum())
    rows = int((b.T_n * (b.U_n + 1)).sum())
    line = {"metric": "full (unpruned) RNN-T loss fwd+bwd frames(N·T)/sec and peak GB, 1 B200", "value":
            frames / (statistics.mean(ms) / 1000.0), "unit": UNIT, "n_gpus": 1, "steps": K,
            "warmup": max(args.warmup, 3), "ms_per_step": statistics.mean(ms), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16+f32", "data": "synthetic",
            "config": {"workload": "c2 batch, full lattice through the joiner (S = U+1, SURVEY 8(f) f4)",
                       "N": b.N, "V": b.V, "J": b.J, "frames": frames, "joiner_rows": rows,
                       "l2": "flushed between timed steps", "kernels": R.rnnt_version()},
            "peak_gib": torch.cuda.max_memory_allocated() / 2 ** 30 - flush.numel() / 2 ** 30,
            "workspace_gib": ws.numel() / 2 ** 30, "clocks": clk}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, world, rank)
    if args.workload == "dynamic":
        return run_dynamic(args)
    if args.workload == "full":
        return run_full(args)
    import torch
    import paper_2206_13236_b200 as R
    # RNNT_BENCH_FUNCTIONAL_DIST=1 (tests only, never a measurement): every rank on cuda:0 and gloo for
    # the exchange, to exercise the N > 1 code path (sharding, the d_w stream hook, max-over-ranks
    # timing, rank-0 output) on a one-GPU box
    functional = os.environ.get("RNNT_BENCH_FUNCTIONAL_DIST") == "1"
    if functional:
        local = 0
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        if functional:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    cfg, b, name = workload(args, world, rank)
    dev = R.batch_to_device(b, "cuda")
    dims = R.make_dims(b.N, b.T, b.U, b.V, b.J, b.S)
    outs = R.alloc_outputs(dims, "cuda")
    from paper_2206_13236_b200.dist import GradBuffer
    # d_w, d_b and the masked loss sums in one flat buffer: at N = 1 plain stores, at N > 1 one NCCL
    # all_reduce (or NVLS multimem adds) per step
    xmode = "local" if pg is None else ("nccl" if functional else args.exchange)
    gbuf = GradBuffer(b.V, b.J, "cuda", mode=xmode)
    outs["d_w"], outs["d_b"] = gbuf.d_w, gbuf.d_b
    ws = torch.empty(R.rnnt_workspace_bytes(dims), dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2
    # the step runs on a high-priority stream (its side streams are lowest priority)
    stream = R.critical_stream() if not args.no_priority else torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    def step(inp, overlap=True):
        # the exchange runs on the d_w stream (R.step exchange=): overlaps the d_enc / d_dec kernels
        outs["status"].zero_()
        R.step(inp["am"], inp["lm"], inp["symbols"], inp["boundary"], inp["enc_proj"], inp["dec_proj"],
               inp["w_out"], inp["b_out"], b.S, out=outs, workspace=ws, exchange=gbuf, overlap=overlap)

    ids = R.kernel_ids()
    kname = args.profile_kernel if args.profile_kernel != "auto" else "joiner_fwd_gemm"
    kid = ids[kname]

    for _ in range(args.warmup):
        step(dev)
    torch.cuda.synchronize()
    if pg is not None:
        pg.barrier()
    torch.cuda.reset_peak_memory_stats()
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for a, c in kev:   # materialise the event handles
        a.record(); c.record()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = R.rnnt_launch_count()
    torch.cuda.synchronize()
    if pg is not None:
        pg.barrier()
    for i in range(K):
        flush.zero_()                       # evict L2 between timed steps
        R.rnnt_profile_kernel(kid, kev[i][0], kev[i][1])
        ev[i][0].record(stream)
        step(dev)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    R.rnnt_profile_kernel(0)
    launches = R.rnnt_launch_count() - launches0
    if pg is not None:
        pg.barrier()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(c) for a, c in ev]
    eager_ms = list(step_ms)

    # The same step captured once as a CUDA graph (all streams: the side-stream branches become graph
    # branches; at N > 1 the NCCL all_reduce is captured too) and replayed: what a training loop on
    # fixed-shape batches runs.  Same timing rules (events on the stream, L2 flushed between replays
    # outside the events, barrier before the timed replays, max over ranks).
    graph = None
    graph_err = None
    if not args.no_graph and not functional:
        try:
            graph = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream()
            cs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(cs):
                step(dev)
            torch.cuda.current_stream().wait_stream(cs)
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=stream):
                step(dev)
            torch.cuda.synchronize()
            for _ in range(max(3, args.warmup)):
                graph.replay()
            torch.cuda.synchronize()
            gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
            clocks = Clocks(local)
            clocks.start()
            time.sleep(0.3)
            if pg is not None:
                pg.barrier()
            torch.cuda.synchronize()
            for i in range(K):
                flush.zero_()
                gev[i][0].record(stream)
                graph.replay()
                gev[i][1].record(stream)
            torch.cuda.synchronize()
            clk = clocks.stop()
            step_ms = [a.elapsed_time(c) for a, c in gev]
        except Exception as e:   # keep the eager numbers
            graph, graph_err = None, f"{type(e).__name__}: {e}"[:200]
            step_ms = eager_ms
    kern_ms = [a.elapsed_time(c) for a, c in kev]
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device="cuda")
    if pg is not None:
        pg.all_reduce(tot, op=pg.ReduceOp.MAX)
    ms_per_step = float(tot.item()) / K
    frames_local = int(b.T_n.sum())
    fr = torch.tensor([frames_local], dtype=torch.float64, device="cuda")
    if pg is not None:
        pg.all_reduce(fr)
    frames = float(fr.item())
    value = frames / (ms_per_step / 1000.0)
    peak_gib = torch.cuda.max_memory_allocated() / 2 ** 30
    # inputs+outputs+workspace actually held by the step (the flush buffer excluded)
    step_gib = (peak_gib - flush.numel() / 2 ** 30)

    # Per-kernel times, each kernel bracketed by CUDA events on its launch stream (rnnt_profile_kernel)
    # over a few extra steps (same workload, L2 flushed between steps):
    #   live        -- in the timed configuration (side streams overlapping, so a kernel may share
    #                  the SMs with another one and its time stretches);
    #   standalone  -- the same step with every call serialised on one stream (overlap=False): each
    #                  kernel has the GPU to itself, as in an ncu launch list but warm.
    # Each kernel's roofline ("achieved", "frac") uses its live time over the timed configuration, with
    # the standalone figures next to it; the line's "roofline" is the kernel with the largest
    # standalone share of the (serial) step.
    hbm, tfl, src = peaks()

    def time_kernels(overlap, reps=5):
        out = {}
        for kn in PROFILED:
            if kn not in ids:
                continue
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
            for a, c in evs:
                a.record(); c.record()
            torch.cuda.synchronize()
            for a, c in evs:
                flush.zero_()
                R.rnnt_profile_kernel(ids[kn], a, c)
                step(dev, overlap=overlap)
            torch.cuda.synchronize()
            R.rnnt_profile_kernel(0)
            out[kn] = statistics.mean(a.elapsed_time(c) for a, c in evs)
        return out

    live_ms = time_kernels(True)
    live_ms[kname] = statistics.mean(kern_ms)
    alone_ms = {} if args.no_standalone else time_kernels(False)
    # the serial step itself (for the kernels' shares)
    serial_ms = None
    if alone_ms:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(5):
            flush.zero_()
            e0.record(stream)
            step(dev, overlap=False)
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        serial_ms = statistics.mean(ts)
    step_mean = statistics.mean(step_ms)
    chain = int((b.T_n + b.U_n).max())          # longest anti-diagonal chain (simple lattice)
    kernels = {}
    for kn, lms in live_ms.items():
        ams = alone_ms.get(kn)
        if kn in LATENCY_BOUND:
            r = {"kernel": kn, "bound": "latency", "achieved": lms * 1e6 / chain, "unit": "ns/diagonal",
                 "frac": None, "kernel_ms": lms, "chain_steps": chain}
        else:
            r = roofline(kn, b, lms, hbm, tfl)
            if ams:
                ra = roofline(kn, b, ams, hbm, tfl)
                r["standalone_achieved"], r["standalone_frac"] = ra["achieved"], ra["frac"]
        r["live_ms"] = lms
        r["standalone_ms"] = ams
        r["share_of_step"] = (ams / serial_ms) if (ams and serial_ms) else (lms / step_mean)
        kernels[kn] = r
    dom = max((k for k in kernels if k not in LATENCY_BOUND), key=lambda k: kernels[k]["share_of_step"])
    roof = dict(kernels[dom])
    traffic, tsrc = ncu_traffic(dom, cfg)
    roof.update({"traffic": traffic, "traffic_source": tsrc, "peak_source": src})

    # end-to-end: host pinned inputs -> device, step, loss -> host, all inside the timed region.
    # Double-buffered like a training loop: the H2D copy of step i+1 (copy stream) overlaps the
    # compute of step i; every step still carries its own full H2D and D2H.  With a CUDA graph, one
    # graph per input buffer set.
    e2e = None
    if not args.no_e2e:
        # page-locked buffers from torch's pinned allocator (cudaHostAlloc): measured 54.6 GB/s H2D on the
        # GPU box, against 22 GB/s from tensor.pin_memory() (tools/h2d_bw.py)
        def pinned(t):
            o = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            o.copy_(t)
            return o

        host = {k: pinned(v.cpu()) for k, v in dev.items()}
        bufs = [dev, {k: v.clone() for k, v in dev.items()}]
        # the per-utterance valid rows of the padded inputs, packed once in pinned host memory: each
        # step sends exactly those bytes (one H2D per tensor) and scatters them into the padded device
        # layout (padded input contents are never read, include/rnnt.h)
        rowsof = {"am": b.T_n, "enc_proj": b.T_n, "lm": b.U_n + 1, "dec_proj": b.U_n + 1}
        packed, pidx = {}, {}
        for tname, lens in rowsof.items():
            full_ = host[tname]
            P_ = full_.shape[1]
            idx = np.concatenate([n * P_ + np.arange(int(lens[n])) for n in range(b.N)])
            flat = full_.view(-1, full_.shape[2])
            packed[tname] = pinned(flat[torch.from_numpy(idx)].contiguous())
            pidx[tname] = torch.from_numpy(idx).cuda()
        dpacked = [{t: torch.empty_like(packed[t], device="cuda") for t in packed} for _ in range(2)]
        small = [k for k in host if k not in rowsof and k not in ("w_out", "b_out")]
        h2d = sum(v.numel() * v.element_size() for v in packed.values()) + \
            sum(host[k].numel() * host[k].element_size() for k in small)
        loss_host = torch.empty(2, b.N, dtype=torch.float32, pin_memory=True)
        d2h = loss_host.numel() * 4
        graphs = [graph, None]
        if graph is not None:
            try:
                g1 = torch.cuda.CUDAGraph()
                cs = torch.cuda.Stream()
                cs.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(cs):
                    step(bufs[1])
                torch.cuda.current_stream().wait_stream(cs)
                torch.cuda.synchronize()
                with torch.cuda.graph(g1, stream=stream):
                    step(bufs[1])
                torch.cuda.synchronize()
                graphs[1] = g1
            except Exception:
                graphs = [None, None]
        ncs = max(1, args.copy_streams)
        copy_streams = [torch.cuda.Stream() for _ in range(ncs)]
        copy_stream = copy_streams[0]
        copied = [[torch.cuda.Event() for _ in range(ncs)] for _ in range(2)]
        freed = [torch.cuda.Event(), torch.cuda.Event()]
        # the packed tensors dealt to the copy streams by size (largest first, to the least loaded stream)
        load_, deal = [0] * ncs, {}
        for tname in sorted(packed, key=lambda t: -packed[t].numel()):
            j = load_.index(min(load_))
            deal[tname] = j
            load_[j] += packed[tname].numel()

        def run(nsteps):
            for i in range(nsteps):
                k = i & 1
                for j, cs_ in enumerate(copy_streams):
                    with torch.cuda.stream(cs_):
                        cs_.wait_event(freed[k])              # step i-2 finished reading buffer set k
                        if j == 0:
                            for tname in small:
                                bufs[k][tname].copy_(host[tname], non_blocking=True)
                        for tname in packed:
                            if deal[tname] == j:
                                dpacked[k][tname].copy_(packed[tname], non_blocking=True)
                        copied[k][j].record(cs_)
                for j in range(ncs):
                    stream.wait_event(copied[k][j])
                # the scatter into the padded layout runs on the step's stream, just before it: on the
                # copy stream it would wait for SMs behind the previous step's persistent kernels and
                # stall the copy engine's pipeline
                with torch.cuda.stream(stream):
                    for tname in packed:
                        dst = bufs[k][tname]
                        dst.view(-1, dst.shape[2]).index_copy_(0, pidx[tname], dpacked[k][tname])
                if graphs[k] is not None:
                    graphs[k].replay()
                else:
                    step(bufs[k])
                freed[k].record(stream)
                loss_host[0].copy_(outs["loss_simple"], non_blocking=True)
                loss_host[1].copy_(outs["loss_pruned"], non_blocking=True)

        for ev_ in freed:
            ev_.record(stream)
        run(max(2, args.warmup))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for ev_ in freed:
            ev_.record(stream)
        e0.record(stream)
        for cs_ in copy_streams:
            cs_.wait_stream(stream)
        run(K)
        e1.record(stream)
        torch.cuda.synchronize()
        et = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        if pg is not None:
            pg.all_reduce(et, op=pg.ReduceOp.MAX)
        e_ms = float(et.item()) / K
        e2e = {"value": frames / (e_ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e_ms,
               "pipelining": "H2D of step i+1 overlaps compute of step i (two input buffer sets); only the "
                             "valid rows of each utterance are sent, scattered into the padded layout on device",
               "copy_streams": ncs,
               "execution": "cuda_graph" if graphs[0] is not None else "eager"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        pool = OraclePool(cfg, rank)
        v, f, nu, el = pool.run(args.cpu_seconds, b.N)
        pool.close()
        cpu = {"value": v, "unit": UNIT, "cores": pool.cores, "kind": "oracle",
               "sample": f"{nu} utterance evaluations rotating over the {b.N} utterances of the same batch "
                         f"({f} frames), full fwd+bwd oracle path, {el:.1f}s wall, fp64 numpy, a process pool "
                         f"over utterances on {pool.cores} cores with BLAS limited to 1 thread per process",
               "host_cpu_count": os.cpu_count(), "host_affinity": pool.cores}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "bf16+f32", "data": "synthetic",
                "config": {"workload": name, "N_per_gpu": b.N, "V": b.V, "J": b.J, "S": b.S,
                           "frames": int(frames), "frames_per_gpu": frames_local,
                           "padded_frames_per_gpu": int(b.N * b.T),
                           "l2": "flushed between timed steps (256 MiB write, outside the timed events)",
                           "kernels": R.rnnt_version()},
                "peak_gib": step_gib, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "kernels": {k: {kk: v.get(kk) for kk in ("bound", "achieved", "unit", "frac", "live_ms",
                                                          "standalone_ms", "standalone_frac", "share_of_step")}
                            for k, v in kernels.items()},
                "serial_ms_per_step": serial_ms, "exchange": xmode,
                "gpu_launches": int(launches), "clocks": clk,
                "execution": "cuda_graph" if graph is not None else "eager",
                "eager_ms_per_step": statistics.mean(eager_ms), "graph_error": graph_err,
                "step_ms": {"median": statistics.median(step_ms), "p10": float(np.percentile(step_ms, 10)),
                            "p90": float(np.percentile(step_ms, 90)), "min": min(step_ms), "max": max(step_ms)},
                "workspace_gib": R.rnnt_workspace_bytes(dims) / 2 ** 30}
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
