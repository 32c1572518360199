"""bench.py -- BitDecoding decode hot path on B200: quantized-KV decode attention.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C2|C5|C3|C1|C2w2|C2b4|C4|C4b2]
                    [--impl ours|reference] [--no-cpu-baseline] [--extra]

Prints ONE JSON line (rank 0).  The metric is BASELINE.json's: decode-attention
latency and HBM GB/s on quantized-KV bytes.  ``value`` = quantized-KV bytes
read per step (KVCache::memory() payload + params, kvcache.cpp:330-345; the
SURVEY.md 8(d) model) summed over all ranks / max-over-ranks device time of the
K timed steps.  A "step" is one ``decode_step`` (attention.cpp:164-242) of the
whole batch: append of the new token, residual + split-KV packed attention,
LSE combine, commit (a full residual is quantized+packed inside the step).

Default workload (N=1): BASELINE.json configs[1] = C2, LLaMA-3.1-8B GQA
(32 q / 8 KV heads, d 128), 2-bit KV (KChannel K, group 128, W_n 4 -> N_r 256),
batch 8, 32K context.  L2: every workload rotates across >= 2 cache replicas
whose combined quantized bytes exceed 2x L2, so each step reads its replica
from HBM (no flush kernel inside the timed region).

--gpus N > 1 (torchrun, one process per GPU, NCCL): C2/C3/C1 are weak-scaled
(each rank owns its own batch of sequences; no data-path collective).  C5 is
sequence-split (strong scaling): each rank attends a contiguous block range of
the 128K context and the normalized (o, lse) partials are all-gathered over
NCCL and LSE-merged (combine, attention.cpp:142-162).

--impl reference: the reference's own CPU engine (oracle/_ref, the unmodified
/root/reference/proj sources compiled out-of-tree) timed through its own
run_bench (bench.cpp:80-210) on this host's cores, same workload and metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

D = 128
WORKLOADS = {
    "C1": dict(batch=1, hq=32, hkv=8, bits=4, warp_n=4, g=128, seq=4096,
               desc="LLaMA-3.1-8B decode attn, b1, 32q/8kv, d128, 4-bit g128 N_r128, 4K"),
    "C2": dict(batch=8, hq=32, hkv=8, bits=2, warp_n=4, g=128, seq=32768,
               desc="LLaMA-3.1-8B decode attn, b8, 32q/8kv, d128, 2-bit g128 N_r256, 32K"),
    "C3": dict(batch=32, hq=32, hkv=32, bits=4, warp_n=4, g=128, seq=8192,
               desc="LLaMA-2-7B MHA decode attn, b32, 32q/32kv, d128, 4-bit g128 N_r128, 8K"),
    "C5": dict(batch=1, hq=32, hkv=8, bits=4, warp_n=4, g=128, seq=131072,
               desc="LLaMA-3.1-8B decode attn, b1, 32q/8kv, d128, 4-bit g128 N_r128, 128K"),
    # C2 with the 128-token fp16 residual of configs[0] ("same shape"): 2-bit
    # at W_n = 2 gives N_r = 128 (layout.cpp:74-77)
    "C2w2": dict(batch=8, hq=32, hkv=8, bits=2, warp_n=2, g=128, seq=32768,
                 desc="LLaMA-3.1-8B decode attn, b8, 32q/8kv, d128, 2-bit g128 N_r128 (W_n 2), 32K"),
    # the north-star statement's 4-bit case at the C2 shape (not a BASELINE
    # config): LLaMA-3.1-8B, 4-bit, batch 8, 32K
    "C2b4": dict(batch=8, hq=32, hkv=8, bits=4, warp_n=4, g=128, seq=32768,
                 desc="LLaMA-3.1-8B decode attn, b8, 32q/8kv, d128, 4-bit g128 N_r128, 32K"),
    # quantize-and-pack throughput (BASELINE configs[3]): prefill of 32K fp16
    # K/V tokens x 8 KV heads into the 4-bit / 2-bit layouts
    "C4": dict(batch=1, hq=32, hkv=8, bits=4, warp_n=4, g=128, seq=32768, qpack=True,
               desc="qpack: 32K fp16 K/V tokens x 8 KV heads, d128 -> 4-bit g128 N_r128"),
    "C4b2": dict(batch=1, hq=32, hkv=8, bits=2, warp_n=4, g=128, seq=32768, qpack=True,
                 desc="qpack: 32K fp16 K/V tokens x 8 KV heads, d128 -> 2-bit g128 N_r256"),
}
QPACK_METRIC = "quantize-and-pack throughput (GB/s of fp16 read + packed written), C4"
METRIC = ("decode-attn latency (µs) & HBM GB/s on quantized KV vs 8 TB/s, 4/2-bit, "
          "32K–128K")
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        for k in ("hbm_gbs", "hbm_GBps", "hbm_copy_gbs"):
            if k in j:
                return float(j[k]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        pass
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


def qbytes_model(w, seq=None):
    """packed payload + params bytes of all cells."""
    n_r = 8 * w["warp_n"] * (16 // w["bits"])
    seq = w["seq"] if seq is None else seq
    plen = seq - seq % n_r
    cells = w["batch"] * w["hkv"]
    return cells * (2 * plen * D * w["bits"] // 8 + 4 * D * plen // w["g"] + 4 * plen * D // w["g"])


# ----------------------------------------------------------------- dist
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class Clocks:
    """nvidia-smi clock / throttle sampling during the measured region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# -------------------------------------------------------------- our arm
def run_ours(args, w, world, rank, local):
    import torch
    import torch.distributed as dist
    from paper_2503_18773_b200 import bitkv as bk
    from paper_2503_18773_b200 import sharding

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    seq_split = args.workload == "C5" and world > 1
    # C3 at N > 1: KV-head sharding (BASELINE configs[2]); rank p owns KV
    # heads [p*hkv/N, (p+1)*hkv/N) and their query heads, no data-path
    # communication (sharding.head_range)
    head_shard = args.workload == "C3" and world > 1
    if head_shard:
        h_lo, h_hi = sharding.head_range(w["hkv"], world, rank)
        ng = w["hq"] // w["hkv"]
        w = dict(w, hkv=h_hi - h_lo, hq=(h_hi - h_lo) * ng)
    props = torch.cuda.get_device_properties(dev)
    l2 = getattr(props, "L2_cache_size", 126 * 2**20)
    spec = bk.QuantSpec(w["bits"], bk.QuantAxis.KChannel, w["g"])
    n_r = bk.residual_block_size(w["bits"], w["warp_n"])
    cfg = bk.AttentionConfig(batch=w["batch"], heads_q=w["hq"], heads_kv=w["hkv"], head_dim=D,
                             tile_m=max(1, w["hq"] // w["hkv"]), tile_n=64, num_splits=4,
                             warp_n=w["warp_n"])
    # sequence split: this rank's block range of the prefilled context
    if seq_split:
        nblk = w["seq"] // n_r
        blk_lo, blk_hi = sharding.block_range(nblk, world, rank)
        local_seq = (blk_hi - blk_lo) * n_r + (w["seq"] % n_r if rank == world - 1 else 0)
    else:
        local_seq = w["seq"]
    per_rep = qbytes_model(w, local_seq)
    n_rep = max(2, -(-2 * l2 // max(per_rep, 1)))
    k_iso = min(args.steps, 40)  # event-bracketed (isolated) kernel timing pass
    headroom = args.warmup + args.steps + args.e2e_steps + k_iso + 2 * n_r
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    reps = []
    t_pref = []
    for _ in range(n_rep):
        c = bk.KVCache(w["batch"], w["hkv"], D, w["warp_n"], spec, max_tokens=local_seq + headroom,
                       device=local)
        k = torch.randn((w["batch"], w["hkv"], local_seq, D), generator=gen, device=dev,
                        dtype=torch.float16)
        v = torch.randn((w["batch"], w["hkv"], local_seq, D), generator=gen, device=dev,
                        dtype=torch.float16)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c.prefill_all(k, v)
        e1.record()
        torch.cuda.synchronize()
        t_pref.append(e0.elapsed_time(e1))
        del k, v
        reps.append(c)
    torch.cuda.empty_cache()
    K, W = args.steps, args.warmup
    NQ = K + W + k_iso
    qs = torch.randn((NQ, w["batch"], w["hq"], D), generator=gen, device=dev).half()
    kns = torch.randn((NQ, w["batch"], w["hkv"], D), generator=gen, device=dev).half()
    vns = torch.randn((NQ, w["batch"], w["hkv"], D), generator=gen, device=dev).half()
    q = torch.empty_like(qs[0])
    kn = torch.empty_like(kns[0])
    vn = torch.empty_like(vns[0])
    out = torch.empty((w["batch"], w["hq"], D), device=dev, dtype=torch.float32)
    lse = torch.empty((w["batch"], w["hq"]), device=dev, dtype=torch.float32)
    steppers = [bk.DecodeStepper(c, cfg, q, kn, vn, out) for c in reps]
    rows = w["batch"] * w["hq"]
    comm = None
    if seq_split:  # the exchange: peer-memory merge kernel (default) or NCCL all-gather
        comm = (sharding.PeerSeqSplit(world, rank, rows, D, dev) if args.exchange == "p2p"
                else sharding.SeqSplitComm(world, rows, D, dev))

    def qbytes(r):
        return sum(r.memory().__dict__[f] for f in
                   ("k_packed_payload_bytes", "v_packed_payload_bytes", "params_bytes"))

    # quantized bytes each step reads, tracked on the host without a C-ABI
    # call per step: a replica's packed segment grows by one block per cell
    # when its residual window fills (every cell steps in lockstep)
    cells = w["batch"] * w["hkv"]
    blk0 = [r.packed_len(0, 0) // n_r for r in reps]
    res0 = [r.res_len(0, 0) for r in reps]
    per_blk = [qbytes(r) // max(1, cells * b) for r, b in zip(reps, blk0)]
    steps_done = [0] * n_rep
    for s_ in steppers:
        s_.prebind(qs, kns, vns)

    def one_step(i):
        # inputs of every step are preloaded in HBM (qs/kns/vns slices): the
        # timed region launches only the decode path's own kernels
        j = i % n_rep
        r = reps[j]
        if seq_split:
            last = rank == world - 1
            if args.exchange == "p2p":
                o_s, lse_s = comm.next_slot()
                o_s, lse_s = o_s.view(w["batch"], w["hq"], D), lse_s.view(w["batch"], w["hq"])
            else:
                o_s, lse_s = comm.o, comm.lse
            bk.decode_partial(r, cfg, qs[i], kns[i] if last else None,
                              vns[i] if last else None, 0, 1 << 30, out=o_s, lse=lse_s)
            comm.merge(out)
            return qbytes(r)
        nbytes = cells * (blk0[j] + (res0[j] + steps_done[j]) // n_r) * per_blk[j]
        steppers[j].step_pre(i)
        steps_done[j] += 1
        return nbytes

    # soak (untimed, no append): keeps clocks up while nvidia-smi samples
    clocks = Clocks(local)
    clocks.start()
    t_end = time.time() + args.soak
    while time.time() < t_end:
        for r in reps:
            bk.decode_partial(r, cfg, q, None, None, 0, 1 << 30, out=out, lse=lse)
        torch.cuda.synchronize()
    for i in range(W):
        one_step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    n_launch0 = sum(r.launch_count() for r in reps)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    bytes_total = 0
    ev0.record()
    for i in range(W, W + K):
        bytes_total += one_step(i)
    ev1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    n_launched = sum(r.launch_count() for r in reps) - n_launch0 + (K if seq_split else 0)
    if not seq_split:  # the host-side byte tracking agrees with the cache
        for j, r in enumerate(reps):
            assert qbytes(r) == cells * (blk0[j] + (res0[j] + steps_done[j]) // n_r) * per_blk[j]
    # isolated kernel timing: CUDA events bracket every attention launch (this
    # serializes the launches, so it runs after the timed region)
    for r in reps:
        r.profile_begin()
    for i in range(W + K, W + K + k_iso):
        one_step(i)
    torch.cuda.synchronize()
    kern_ms, launches = 0.0, 0
    for r in reps:
        a, b = r.profile_end()
        kern_ms += a
        launches += b

    # e2e through the public host API (host fp32 in, host fp32 out; copies inside)
    import numpy as np
    e2e_ms = None
    h2d = d2h = 0
    if not seq_split and args.e2e_steps > 0:
        hq = np.random.default_rng(rank).standard_normal(
            (args.e2e_steps, w["batch"], w["hq"], D)).astype(np.float16).astype(np.float32)
        hk = np.random.default_rng(rank + 1).standard_normal(
            (args.e2e_steps, w["batch"], w["hkv"], D)).astype(np.float16).astype(np.float32)
        hv = np.random.default_rng(rank + 2).standard_normal(
            (args.e2e_steps, w["batch"], w["hkv"], D)).astype(np.float16).astype(np.float32)
        hout = np.empty((w["batch"], w["hq"], D), np.float32)  # reused output (decode_step(out=))
        bk.decode_step(reps[0], cfg, hq[0], hk[0], hv[0], out=hout)  # staging allocation
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e2e_bytes = 0
        e2e_s = 0.0
        for i in range(args.e2e_steps):
            r = reps[i % n_rep]
            # the quantized bytes this step attends (read before the call:
            # the step itself may flush a block); outside the timed call
            e2e_bytes += sum(r.memory().__dict__[f] for f in
                             ("k_packed_payload_bytes", "v_packed_payload_bytes",
                              "params_bytes"))
            t0 = time.perf_counter()
            res = bk.decode_step(r, cfg, hq[i], hk[i], hv[i], out=hout)
            e2e_s += time.perf_counter() - t0
        e2e_ms = e2e_s * 1e3
        assert np.isfinite(res.data).all()
        # H2D: the step's q/k_new/v_new as fp16 (converted on the host);
        # D2H: the fp32 output, stored by the kernel into pinned host memory
        h2d = (hq[0].size + hk[0].size + hv[0].size) * 2
        d2h = hq[0].size * 4

    # max over ranks, sum of bytes
    t = torch.tensor([ms, e2e_ms or 0.0, kern_ms], dtype=torch.float64, device=dev)
    b = torch.tensor([float(bytes_total)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if not seq_split:
            dist.all_reduce(b, op=dist.ReduceOp.SUM)
    ms, e2e_ms_max, _ = t.tolist()
    total_bytes = b.item() if not seq_split else qbytes_model(w) * K
    if rank != 0:
        return None
    gbs = total_bytes / (ms * 1e-3) / 1e9
    peak, peak_src = peak_hbm()
    # steady state: one attention launch per step, back to back (PDL-overlapped)
    per_launch_bytes = bytes_total / K
    step_ms = ms / K
    achieved = per_launch_bytes / (step_ms * 1e-3) / 1e9
    kern_avg_ms = kern_ms / max(launches, 1)
    iso = per_launch_bytes / (kern_avg_ms * 1e-3) / 1e9 if launches else None
    res = {
        "metric": METRIC, "value": round(gbs, 1), "unit": "GB/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": round(ms / K, 5),
        "latency_us": round(ms / K * 1e3, 2), "higher_is_better": True,
        "scaling": "strong" if (seq_split or head_shard) else "weak", "vs_baseline": None,
        "dtype": f"u{w['bits']} codes -> fp16 MMA, fp32 accumulate", "data": "synthetic",
        "config": {"workload": f"{args.workload}: {w['desc']}", "batch_per_gpu": w["batch"],
                   "global_batch": w["batch"] * (1 if (seq_split or head_shard) else world),
                   "seq_len": w["seq"], "bits": w["bits"], "group_size": w["g"],
                   "warp_n": w["warp_n"], "n_r": n_r,
                   "parallelism": ((f"seq-split{world} (peer-memory merge kernel over NVLink)"
                                    if args.exchange == "p2p" else
                                    f"seq-split{world} (NCCL all-gather of (o,lse))") if seq_split
                                   else f"kv-head-shard{world} (no communication)" if head_shard
                                   else (f"dp{world} (independent batches)" if world > 1
                                         else "single GPU")),
                   "l2": f"rotating {n_rep} cache replicas x {per_rep/1e6:.1f} MB quantized "
                         f"(> 2x L2 {l2/2**20:.0f} MiB); inputs larger than L2, no flush",
                   "quantized_bytes_per_step": round(total_bytes / K)},
        "roofline": {"bound": "hbm",
                     "achieved": round(achieved, 1) if achieved else None,
                     "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4) if achieved else None,
                     "peak_source": peak_src,
                     "kernel": "bdk::decode_fast_kernel (stream-K attention over packed "
                               "blocks + residual + in-kernel LSE merge)",
                     "duration": "timed region / attention launches (one per step, "
                                 "back to back with programmatic dependent launch)",
                     "kernel_avg_us": round(step_ms * 1e3, 2),
                     "kernel_isolated_us": round(kern_avg_ms * 1e3, 2),
                     "isolated_achieved": round(iso, 1) if iso else None,
                     "isolated_note": "CUDA events around each launch (no PDL overlap, "
                                      "includes launch latency)",
                     "algorithmic_bytes_per_launch": round(per_launch_bytes),
                     "traffic": load_traffic(args.workload)},
        "e2e": ({"value": round(e2e_bytes_rate(bytes_total / K, args.e2e_steps, e2e_ms_max,
                                               world), 2),
                 "unit": "GB/s", "latency_us": round(e2e_ms_max / args.e2e_steps * 1e3, 1),
                 "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                 "path": "bitkv.decode_step(host fp32 arrays) -> bdk_decode_step_host "
                         "(host F16C convert to pinned fp16, one H2D, decode, fp32 output to "
                         "pinned host memory -- kernel stores when <= 256 KiB, else one D2H "
                         "copy -- sync, copy out)",
                 "clock": "host perf_counter (synchronous call)"}
                if e2e_ms else None),
        "gpu_launches": n_launched,
        "clocks": clk,
        "prefill_ms_per_replica": round(statistics.median(t_pref), 3),
    }
    return res


def e2e_bytes_rate(bytes_per_step, steps, ms, world):
    return bytes_per_step * world * steps / (ms * 1e-3) / 1e9


def load_traffic(workload):
    p = os.path.join(ROOT, "profiles", "ncu_decode_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


# ------------------------------------------------ C4: quantize-and-pack
def qpack_bytes(w):
    """fp16 K/V read + packed words and (scale, zero) params written
    (SURVEY.md 8(d), C4 rows)."""
    n_r = 8 * w["warp_n"] * (16 // w["bits"])
    cells = w["batch"] * w["hkv"]
    plen = w["seq"] - w["seq"] % n_r
    rd = 2 * cells * w["seq"] * D * 2
    wr = cells * (2 * plen * D * w["bits"] // 8 + 4 * D * plen // w["g"] + 4 * plen * D // w["g"])
    return rd, wr


def run_qpack(args, w, world, rank, local):
    """Prefill (KVCache::prefill, kvcache.cpp:155-168) of every cell: one
    fused quantize+pack launch per step into a fresh cache."""
    import torch
    import torch.distributed as dist
    from paper_2503_18773_b200 import bitkv as bk

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    spec = bk.QuantSpec(w["bits"], bk.QuantAxis.KChannel, w["g"])
    gen = torch.Generator(device=dev)
    gen.manual_seed(4321 + rank)
    shape = (w["batch"], w["hkv"], w["seq"], D)
    k = torch.randn(shape, generator=gen, device=dev, dtype=torch.float16)
    v = torch.randn(shape, generator=gen, device=dev, dtype=torch.float16)
    K, W = args.steps, args.warmup
    n_c = min(K, 32)
    caches = [bk.KVCache(w["batch"], w["hkv"], D, w["warp_n"], spec, max_tokens=w["seq"],
                         device=local) for _ in range(n_c)]
    for i in range(W):
        caches[i % n_c].reset()
        caches[i % n_c].prefill_all(k, v)
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    t_end = time.time() + args.soak  # untimed: keeps clocks up while nvidia-smi samples
    while time.time() < t_end:
        for c in caches:
            c.reset()
            c.prefill_all(k, v)
        torch.cuda.synchronize()
    ms, done = 0.0, 0
    n_launch0 = sum(c.launch_count() for c in caches)
    while done < K:
        n = min(n_c, K - done)
        for c in caches[:n]:
            c.reset()  # untimed: the timed region is the prefill launches only
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for c in caches[:n]:
            c.prefill_all(k, v)
        e1.record()
        torch.cuda.synchronize()
        ms += e0.elapsed_time(e1)
        done += n
    clk = clocks.stop()
    n_launched = sum(c.launch_count() for c in caches) - n_launch0
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    rd, wr = qpack_bytes(w)
    mem = caches[0].memory().__dict__
    wr_live = mem["k_packed_payload_bytes"] + mem["v_packed_payload_bytes"] + mem["params_bytes"]
    assert wr_live == wr, (wr_live, wr)
    # e2e: host (pinned) fp16 K/V -> KVCache.prefill_all through the public
    # API: H2D copy of the step's K/V + the qpack launch, synchronized
    kh = k.cpu().pin_memory()
    vh = v.cpu().pin_memory()
    kd, vd = torch.empty_like(k), torch.empty_like(v)
    e2e_steps = max(1, min(5, args.e2e_steps))
    e2e_s = 0.0
    for _ in range(e2e_steps):
        c = caches[0]
        c.reset()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        kd.copy_(kh, non_blocking=True)
        vd.copy_(vh, non_blocking=True)
        c.prefill_all(kd, vd)
        torch.cuda.synchronize()
        e2e_s += time.perf_counter() - t0
    if rank != 0:
        return None
    per_step = (rd + wr)
    gbs = per_step * world * K / (ms * 1e-3) / 1e9
    achieved = per_step / (ms / K * 1e-3) / 1e9
    peak, peak_src = peak_hbm()
    res = {
        "metric": QPACK_METRIC, "value": round(gbs, 1), "unit": "GB/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": round(ms / K, 5),
        "latency_us": round(ms / K * 1e3, 2), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": f"fp16 -> u{w['bits']} codes (bit-exact integer pack)",
        "data": "synthetic",
        "config": {"workload": f"{args.workload}: {w['desc']}", "cells": w["batch"] * w["hkv"],
                   "seq_len": w["seq"], "bits": w["bits"], "group_size": w["g"],
                   "warp_n": w["warp_n"], "parallelism": "single GPU" if world == 1
                   else f"dp{world} (independent caches)",
                   "l2": "inputs 2 x %.0f MB fp16 (> L2), fresh cache per step" % (rd / 2e6),
                   "bytes_read_per_step": rd, "bytes_written_per_step": wr},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "peak_source": peak_src,
                     "kernel": "bdk::prefill_kernel (fused quantize + pack, bdk_qpack.cuh)",
                     "duration": "timed region / prefill launches (events, one launch per step)",
                     "algorithmic_bytes_per_launch": per_step,
                     "traffic": load_traffic(args.workload)},
        "e2e": {"value": round(per_step * e2e_steps / e2e_s / 1e9, 2), "unit": "GB/s",
                "latency_us": round(e2e_s / e2e_steps * 1e6, 1),
                "h2d_bytes_per_step": rd, "d2h_bytes_per_step": 0,
                "path": "pinned host fp16 K/V -> H2D -> KVCache.prefill_all (qpack) -> sync",
                "clock": "host perf_counter"},
        "gpu_launches": n_launched, "clocks": clk, "cpu_baseline": None,
    }
    return res


def cpu_qpack_reference(w):
    """The reference's prefill (single-threaded by construction, bench.cpp:
    132-139) through its own run_bench: (GB/s, seconds, kind, sample)."""
    from oracle import oracle as O
    rd, wr = qpack_bytes(w)
    if O.have_ref():
        r = O.ref_run_bench(mode=0, seq_len=w["seq"], batch=w["batch"], heads_q=w["hq"],
                            heads_kv=w["hkv"], head_dim=D, bits=w["bits"], group_size=w["g"],
                            k_axis=0, num_splits=4, steps=1, seed=0, tile_n=64,
                            warp_n=w["warp_n"])
        sec = r["prefill_seconds"]
        return ((rd + wr) / sec / 1e9, sec, "reference",
                f"reference run_bench prefill_seconds (bench.cpp:132-139), full C4 shape, "
                f"1 thread by construction")
    import numpy as np
    g = O.Gauss(0)
    oc = O.OracleCache(w["batch"], w["hkv"], D, w["warp_n"], w["bits"], 0, w["g"], True,
                       max_tokens=w["seq"])
    ks = [g.rounded(w["seq"] * D).reshape(w["seq"], D) for _ in range(2 * w["hkv"])]
    t0 = time.perf_counter()
    for h in range(w["hkv"]):
        oc.prefill(0, h, ks[2 * h], ks[2 * h + 1])
    sec = time.perf_counter() - t0
    del np
    return ((rd + wr) / sec / 1e9, sec, "port",
            "oracle C restatement prefill, full C4 shape, 1 thread")


# ------------------------------------------------------- CPU reference arm
def cpu_reference(w, steps, warm=1):
    """The unmodified reference engine (oracle/_ref) via its own run_bench,
    or the C restatement (kind "port") when _ref is absent.  Returns
    (GB/s, mean step ms, kind, cores, sample)."""
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    os.environ["BITKV_THREADS"] = str(cores)
    n_r = 8 * w["warp_n"] * (16 // w["bits"])
    qb = qbytes_model(w)
    if O.have_ref():
        r = O.ref_run_bench(mode=1 if w["batch"] > 1 else 0, seq_len=w["seq"], batch=w["batch"],
                            heads_q=w["hq"], heads_kv=w["hkv"], head_dim=D, bits=w["bits"],
                            group_size=w["g"], k_axis=0, num_splits=4, steps=warm + steps,
                            seed=0, tile_n=64, warp_n=w["warp_n"])
        mem = r["memory"]
        qb = mem[0] + mem[1] + mem[2]
        st = r["step_ms"][warm:]
        ms = sum(st) / len(st)
        kind = "reference"
        sample = (f"reference run_bench (bench.cpp:80-210), full {w['seq']}-token shape, "
                  f"{steps} timed decode steps after {warm} warm-up, prefill "
                  f"{r['prefill_seconds']:.2f} s single-threaded; BITKV_THREADS={cores}")
    else:
        import numpy as np
        g = O.Gauss(0)
        oc = O.OracleCache(w["batch"], w["hkv"], D, w["warp_n"], w["bits"], 0, w["g"], True,
                           max_tokens=w["seq"] + steps + warm + n_r)
        for b in range(w["batch"]):
            for h in range(w["hkv"]):
                k = g.rounded(w["seq"] * D).reshape(w["seq"], D)
                v = g.rounded(w["seq"] * D).reshape(w["seq"], D)
                oc.prefill(b, h, k, v)
        times = []
        for s in range(warm + steps):
            q = g.rounded(w["batch"] * w["hq"] * D).reshape(w["batch"], w["hq"], D)
            kn = g.rounded(w["batch"] * w["hkv"] * D).reshape(w["batch"], w["hkv"], D)
            vn = g.rounded(w["batch"] * w["hkv"] * D).reshape(w["batch"], w["hkv"], D)
            t0 = time.perf_counter()
            oc.decode_step(q, kn, vn, threads=cores)
            times.append((time.perf_counter() - t0) * 1e3)
        ms = sum(times[warm:]) / steps
        kind = "port"
        sample = (f"oracle C restatement (oracle/bitkv_oracle.c), full shape, {steps} steps, "
                  f"{cores} threads")
        del np
    return qb / (ms * 1e-3) / 1e9, ms, kind, cores, sample


def run_reference_arm(args, w, world, rank):
    if rank != 0:
        return None
    if w.get("qpack"):
        gbs, sec, kind, sample = cpu_qpack_reference(w)
        return {"impl": "reference", "metric": QPACK_METRIC, "value": round(gbs, 4),
                "unit": "GB/s", "n_gpus": world, "steps": 1, "warmup": 0,
                "ms_per_step": round(sec * 1e3, 3), "latency_us": round(sec * 1e6, 1),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": f"fp32 -> u{w['bits']} codes (CPU)", "data": "synthetic",
                "config": {"workload": f"{args.workload}: {w['desc']}", "seq_len": w["seq"]},
                "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": 1,
                                 "kind": kind, "sample": sample},
                "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
    steps = args.steps
    # bound the run: the reference step at C2/C5 is ~1 s on 8 cores
    est = {"C1": 0.05, "C2": 1.7, "C2b4": 1.7, "C2w2": 1.7, "C3": 5.0, "C5": 0.9}[args.workload] * 8 / (os.cpu_count() or 8)
    cap = max(2, int(150 / max(est, 1e-3)))
    k_run = min(steps, cap)
    gbs, ms, kind, cores, sample = cpu_reference(w, k_run, warm=min(args.warmup, 1))
    if k_run < steps:
        sample += f" (K capped at {k_run} of {steps} to bound the run)"
    line = {"impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s",
            "n_gpus": world, "steps": k_run, "warmup": min(args.warmup, 1),
            "ms_per_step": round(ms, 3), "latency_us": round(ms * 1e3, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": f"u{w['bits']} codes -> fp32 (CPU)", "data": "synthetic",
            "config": {"workload": f"{args.workload}: {w['desc']}", "global_batch": w["batch"],
                       "seq_len": w["seq"]},
            "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": cores,
                             "kind": kind, "sample": sample},
            "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--workload", default="C2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--soak", type=float, default=1.0, help="untimed seconds before timing")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="C5 sequence split: peer-memory merge kernel or NCCL all-gather")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=3)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    w = WORKLOADS[args.workload]
    world, rank, local = dist_env()
    if args.impl == "reference":
        line = run_reference_arm(args, w, world, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    import torch
    import torch.distributed as dist
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        if w.get("qpack"):
            res = run_qpack(args, w, world, rank, local)
            if res is not None and world == 1 and not args.no_cpu_baseline:
                gbs, sec, kind, sample = cpu_qpack_reference(w)
                res["cpu_baseline"] = {"value": round(gbs, 4), "unit": "GB/s", "cores": 1,
                                       "kind": kind, "sample": sample,
                                       "ms_per_step": round(sec * 1e3, 2)}
            if res is not None:
                print(json.dumps(res), flush=True)
            return
        res = run_ours(args, w, world, rank, local)
        if res is not None:
            if world == 1 and not args.no_cpu_baseline:
                gbs, ms, kind, cores, sample = cpu_reference(w, args.cpu_steps)
                res["cpu_baseline"] = {"value": round(gbs, 4), "unit": "GB/s", "cores": cores,
                                       "kind": kind, "sample": sample,
                                       "ms_per_step": round(ms, 2)}
            else:
                res["cpu_baseline"] = None
            print(json.dumps(res), flush=True)
    finally:
        if world > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
