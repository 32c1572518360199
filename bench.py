"""bench.py -- BitDecoding decode hot path on B200: quantized-KV decode attention.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C5|C2|C3|C1|C4|...]
                    [--impl ours|reference] [--quick] [--no-extras] [--no-parity]
                    [--no-cpu-baseline] [--exchange p2p|nccl] [--dry-run]

Prints ONE JSON line (rank 0).  The metric is BASELINE.json's: decode-attention
latency and HBM GB/s on quantized-KV bytes.  ``value`` = quantized-KV bytes
read per step (KVCache::memory() payload + params, kvcache.cpp:330-345; the
SURVEY.md 8(d) model) of the whole job / max-over-ranks device time of the K
timed steps.  A "step" is one ``decode_step`` (attention.cpp:164-242) of the
whole batch: append of the new token, residual + split-KV packed attention,
LSE combine, commit (a residual that fills is quantized+packed inside the step).

Headline workload at every N: BASELINE.json configs[4] = C5, the north-star
case: LLaMA-3.1-8B (32 q / 8 KV heads, d 128), 4-bit KV (KChannel K, group 128,
N_r 128), batch 1, 128K context, fast mode (the throughput kernel).  At N > 1 it
is sequence-split (strong scaling): rank p attends a contiguous block range of
the 128K context and the normalized (o, lse) partials are merged by
``bdk_peer_merge`` -- one kernel per rank that reads the peers' partials over
NVLink peer memory (combine, attention.cpp:142-162); ``--exchange nccl``, or
GPUs without peer access, use the NCCL all-gather + merge kernel instead.

The same line carries (rank 0):
  extras     every other BASELINE config, timed the same way: C2 (2-bit b8 32K),
             C3 (MHA b32 8K; KV-head sharded at N > 1), C1 (4K), C4/C4b2
             (quantize-and-pack), and the precise mode (the reference's 1e-5
             contract) of C5 and C2;
  parity     per config, outside every timed region: the GPU output on the
             reference's own bytes -- run_bench's GaussianSource stream (seed 0,
             bench.cpp:18-35, draw order :116-155) -- against the reference's
             decode_step on the same bytes (oracle/_ref, the unmodified engine):
             max-abs / rel-L2 for the fast and the precise mode; C4: sha256 of
             every packed block against the reference-generated hashes
             (tests/golden/blocks.json);
  cpu_baseline  (N = 1) the reference's decode_step timed in that parity pass on
             all host cores.
L2: every timed workload rotates across >= 2 cache replicas whose combined
quantized bytes exceed 2x L2, so each step reads its replica from HBM.

--gpus N without torchrun re-launches this script under
``torch.distributed.run`` with N ranks (127.0.0.1).  ``--dry-run`` checks that
plumbing on CPU (gloo, no CUDA).

--impl reference: the reference's own CPU engine (oracle/_ref, the unmodified
/root/reference/proj sources compiled out-of-tree) timed through its own
run_bench (bench.cpp:80-210) on this host's cores, same workload, metric and
config; rank 0 only.
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
    # the north-star statement's 4-bit case at the C2 shape (not a BASELINE config)
    "C2b4": dict(batch=8, hq=32, hkv=8, bits=4, warp_n=4, g=128, seq=32768,
                 desc="LLaMA-3.1-8B decode attn, b8, 32q/8kv, d128, 4-bit g128 N_r128, 32K"),
    # quantize-and-pack throughput (BASELINE configs[3]): prefill of 32K fp16
    # K/V tokens x 8 KV heads into the 4-bit / 2-bit layouts
    "C4": dict(batch=1, hq=32, hkv=8, bits=4, warp_n=4, g=128, seq=32768, qpack=True,
               desc="qpack: 32K fp16 K/V tokens x 8 KV heads, d128 -> 4-bit g128 N_r128"),
    "C4b2": dict(batch=1, hq=32, hkv=8, bits=2, warp_n=4, g=128, seq=32768, qpack=True,
                 desc="qpack: 32K fp16 K/V tokens x 8 KV heads, d128 -> 2-bit g128 N_r256"),
}
DEFAULT_WORKLOAD = "C5"
# (workload, mode) pairs reported under "extras" next to the headline
EXTRAS = [("C5", "precise"), ("C2", "fast"), ("C2", "precise"), ("C3", "fast"), ("C1", "fast"),
          ("C4", None), ("C4b2", None)]
# parity on the reference's bytes: decode workloads (C4 is checked by hashes)
PARITY = ["C5", "C2", "C1", "C3"]
# golden block hashes of the C4 flush (tests/golden/make_golden.py BLOCK_CASES)
C4_GOLDEN = {"C4": "c4_flush_4bit_32k", "C4b2": "c4_flush_2bit_32k"}
QPACK_METRIC = "quantize-and-pack throughput (GB/s of fp16 read + packed written), C4"
METRIC = ("decode-attn latency (µs) & HBM GB/s on quantized KV vs 8 TB/s, 4/2-bit, "
          "32K–128K")
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
# stated tolerances: precise = the reference's own bar
# (test_attention.cpp:350-441); fast = the fp16-P kernel
TOL = {"precise": {"max_abs": 1e-5}, "fast": {"max_abs": 2e-3, "rel_l2": 2e-3}}


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


def n_r_of(w):
    return 8 * w["warp_n"] * (16 // w["bits"])


def qbytes_model(w, seq=None, batch=None, hkv=None):
    """packed payload + params bytes of all cells."""
    n_r = n_r_of(w)
    seq = w["seq"] if seq is None else seq
    plen = seq - seq % n_r
    cells = (w["batch"] if batch is None else batch) * (w["hkv"] if hkv is None else hkv)
    return cells * (2 * plen * D * w["bits"] // 8 + 4 * D * plen // w["g"] + 4 * plen * D // w["g"])


def qpack_bytes(w):
    """fp16 K/V read + packed words and (scale, zero) params written
    (SURVEY.md 8(d), C4 rows)."""
    cells = w["batch"] * w["hkv"]
    plen = w["seq"] - w["seq"] % n_r_of(w)
    rd = 2 * cells * w["seq"] * D * 2
    wr = cells * (2 * plen * D * w["bits"] // 8 + 4 * D * plen // w["g"] + 4 * plen * D // w["g"])
    return rd, wr


def split_kind(name, world):
    """How workload `name` is spread over `world` GPUs."""
    if world == 1:
        return "single"
    if name == "C5":
        return "seq"
    if name == "C3":
        return "head"
    return "dp"


def workload_config(name, world):
    """The `config` object -- identical for both arms (the reference arm runs
    the same whole-job workload on the host)."""
    w = WORKLOADS[name]
    kind = split_kind(name, world)
    gb = w["batch"] * (world if kind == "dp" else 1)
    par = {"single": "single GPU",
           "seq": f"seq-split{world} (block ranges per GPU, (o, lse) partials LSE-merged over NVLink)",
           "head": f"kv-head-shard{world} (no communication)",
           "dp": f"dp{world} (independent batches, no communication)"}[kind]
    cfg = {"workload": f"{name}: {w['desc']}", "global_batch": gb, "seq_len": w["seq"],
           "heads_q": w["hq"], "heads_kv": w["hkv"], "head_dim": D, "bits": w["bits"],
           "group_size": w["g"], "warp_n": w["warp_n"], "n_r": n_r_of(w), "parallelism": par}
    if w.get("qpack"):
        rd, wr = qpack_bytes(w)
        cfg["bytes_per_step"] = (rd + wr) * (world if kind == "dp" else 1)
    else:
        cfg["quantized_bytes_per_step"] = qbytes_model(w, batch=gb)
    return cfg


# ----------------------------------------------------------------- dist
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(n):
    """--gpus N outside torchrun: run this script as N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


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


def load_traffic(key):
    p = os.path.join(ROOT, "profiles", "ncu_decode_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(key)
    except Exception:
        return None


def oversubscribed(world):
    """Dev knob BDK_BENCH_OVERSUB=1: more ranks than GPUs share them (rank r
    on GPU r % count, gloo process group) -- exercises the N-rank plumbing,
    the head/sequence split and the peer-memory exchange on one GPU; its
    timings mean nothing."""
    import torch
    return os.environ.get("BDK_BENCH_OVERSUB") == "1" and world > torch.cuda.device_count()


def peer_ok(world, local):
    """True when this GPU can map every peer's memory (P2P over NVLink)."""
    import torch
    if oversubscribed(world):  # every rank's buffers on this GPU: CUDA IPC, no peer link
        return True
    return all(torch.cuda.can_device_access_peer(local, p) for p in range(world) if p != local)


# ----------------------------------------------------- decode (our arm)
def run_decode(args, name, mode, world, rank, local, steps, warmup, e2e_steps, soak,
               sample_clocks=False):
    """Time `steps` decode steps of workload `name` (every rank), return the
    rank-0 result dict (None elsewhere)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2503_18773_b200 import bitkv as bk
    from paper_2503_18773_b200 import sharding

    w = dict(WORKLOADS[name])
    kind = split_kind(name, world)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if kind == "head":
        h_lo, h_hi = sharding.head_range(w["hkv"], world, rank)
        ng = w["hq"] // w["hkv"]
        w.update(hkv=h_hi - h_lo, hq=(h_hi - h_lo) * ng)
    props = torch.cuda.get_device_properties(dev)
    l2 = getattr(props, "L2_cache_size", 126 * 2**20)
    spec = bk.QuantSpec(w["bits"], bk.QuantAxis.KChannel, w["g"])
    n_r = n_r_of(w)
    cfg = bk.AttentionConfig(batch=w["batch"], heads_q=w["hq"], heads_kv=w["hkv"], head_dim=D,
                             tile_m=max(1, w["hq"] // w["hkv"]), tile_n=64, num_splits=4,
                             warp_n=w["warp_n"])
    seq_split = kind == "seq"
    if seq_split:
        nblk = w["seq"] // n_r
        blk_lo, blk_hi = sharding.block_range(nblk, world, rank)
        local_seq = (blk_hi - blk_lo) * n_r + (w["seq"] % n_r if rank == world - 1 else 0)
    else:
        local_seq = w["seq"]
    per_rep = qbytes_model(w, local_seq)
    n_rep = max(2, -(-2 * l2 // max(per_rep, 1)))
    k_iso = min(steps, 40)  # event-bracketed (isolated) kernel timing pass
    headroom = warmup + steps + e2e_steps + k_iso + 2 * n_r
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    reps, t_pref = [], []
    for _ in range(n_rep):
        c = bk.KVCache(w["batch"], w["hkv"], D, w["warp_n"], spec, max_tokens=local_seq + headroom,
                       device=local, precise=(mode == "precise"))
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
    K, W = steps, warmup
    NQ = K + W + k_iso
    qs = torch.randn((NQ, w["batch"], w["hq"], D), generator=gen, device=dev).half()
    kns = torch.randn((NQ, w["batch"], w["hkv"], D), generator=gen, device=dev).half()
    vns = torch.randn((NQ, w["batch"], w["hkv"], D), generator=gen, device=dev).half()
    q, kn, vn = torch.empty_like(qs[0]), torch.empty_like(kns[0]), torch.empty_like(vns[0])
    out = torch.empty((w["batch"], w["hq"], D), device=dev, dtype=torch.float32)
    lse = torch.empty((w["batch"], w["hq"]), device=dev, dtype=torch.float32)
    steppers = [bk.DecodeStepper(c, cfg, q, kn, vn, out) for c in reps]
    rows = w["batch"] * w["hq"]
    comm, exchange = None, None
    if seq_split:
        exchange = args.exchange if (args.exchange == "nccl" or peer_ok(world, local)) else "nccl"
        comm = (sharding.PeerSeqSplit(world, rank, rows, D, dev) if exchange == "p2p"
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
            if exchange == "p2p":
                o_s, lse_s = comm.next_slot()
                o_s, lse_s = o_s.view(w["batch"], w["hq"], D), lse_s.view(w["batch"], w["hq"])
            else:
                o_s, lse_s = comm.o.view(w["batch"], w["hq"], D), comm.lse.view(w["batch"], w["hq"])
            bk.decode_partial(r, cfg, qs[i], kns[i] if last else None,
                              vns[i] if last else None, 0, 1 << 30, out=o_s, lse=lse_s)
            comm.merge(out)
            return qbytes(r)
        nbytes = cells * (blk0[j] + (res0[j] + steps_done[j]) // n_r) * per_blk[j]
        steppers[j].step_pre(i)
        steps_done[j] += 1
        return nbytes

    clocks = Clocks(local) if sample_clocks else None
    if clocks:
        clocks.start()
    t_end = time.time() + soak  # untimed, no append: keeps clocks up while nvidia-smi samples
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
    clk = clocks.stop() if clocks else None
    ms = ev0.elapsed_time(ev1)
    n_launched = sum(r.launch_count() for r in reps) - n_launch0 + (K if seq_split else 0)
    if not seq_split:  # the host-side byte tracking agrees with the cache
        for j, r in enumerate(reps):
            assert qbytes(r) == cells * (blk0[j] + (res0[j] + steps_done[j]) // n_r) * per_blk[j]
    if seq_split and exchange == "p2p":
        comm.check()
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

    # e2e through the public API: host fp32 in (pinned for the seq split),
    # host fp32 out, copies inside the timed call
    e2e_ms, h2d, d2h, e2e_bytes = None, 0, 0, 0
    if e2e_steps > 0:
        rng = np.random.default_rng(rank)
        hq = rng.standard_normal((e2e_steps, w["batch"], w["hq"], D)).astype(np.float16).astype(
            np.float32)
        hk = rng.standard_normal((e2e_steps, w["batch"], w["hkv"], D)).astype(np.float16).astype(
            np.float32)
        hv = rng.standard_normal((e2e_steps, w["batch"], w["hkv"], D)).astype(np.float16).astype(
            np.float32)
        hout = np.empty((w["batch"], w["hq"], D), np.float32)  # reused output (decode_step(out=))
        if seq_split:
            last = rank == world - 1
            hq_p = torch.from_numpy(hq).half().pin_memory()
            hk_p = torch.from_numpy(hk).half().pin_memory()
            hv_p = torch.from_numpy(hv).half().pin_memory()
            hout_p = torch.empty((w["batch"], w["hq"], D), dtype=torch.float32).pin_memory()
            qd, kd, vd = torch.empty_like(qs[0]), torch.empty_like(kns[0]), torch.empty_like(vns[0])

            def e2e_one(i):
                r = reps[0]
                qd.copy_(hq_p[i], non_blocking=True)
                if last:
                    kd.copy_(hk_p[i], non_blocking=True)
                    vd.copy_(hv_p[i], non_blocking=True)
                o_s, lse_s = (comm.next_slot() if exchange == "p2p" else (comm.o, comm.lse))
                bk.decode_partial(r, cfg, qd, kd if last else None, vd if last else None, 0,
                                  1 << 30, out=o_s.view(w["batch"], w["hq"], D),
                                  lse=lse_s.view(w["batch"], w["hq"]))
                comm.merge(out)
                hout_p.copy_(out, non_blocking=True)
                torch.cuda.synchronize()
            e2e_one(0)
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            for i in range(e2e_steps):
                e2e_one(i)
            e2e_s = time.perf_counter() - t0
            e2e_bytes = qbytes_model(w) * e2e_steps
            # rank 0's copies: fp16 q (+ k_new/v_new on the last rank), fp32 out
            h2d = (hq[0].size + ((hk[0].size + hv[0].size) if last else 0)) * 2
            d2h = hq[0].size * 4
            res_e2e = hout_p.numpy()
        else:
            bk.decode_step(reps[0], cfg, hq[0], hk[0], hv[0], out=hout)  # staging allocation
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e2e_s = 0.0
            for i in range(e2e_steps):
                r = reps[i % n_rep]
                # the quantized bytes this step attends (read before the call:
                # the step itself may flush a block); outside the timed call
                e2e_bytes += qbytes(r)
                t0 = time.perf_counter()
                res_e2e = bk.decode_step(r, cfg, hq[i], hk[i], hv[i], out=hout).data
                e2e_s += time.perf_counter() - t0
            # H2D: the step's q/k_new/v_new as fp16 (converted on the host);
            # D2H: the fp32 output, stored by the kernel into pinned host memory
            h2d = (hq[0].size + hk[0].size + hv[0].size) * 2
            d2h = hq[0].size * 4
        e2e_ms = e2e_s * 1e3
        assert np.isfinite(res_e2e).all()

    # max over ranks (times), sum over ranks (bytes, weak/head shard)
    t = torch.tensor([ms, e2e_ms or 0.0, kern_ms], dtype=torch.float64, device=dev)
    b = torch.tensor([float(bytes_total), float(e2e_bytes)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if not seq_split:
            dist.all_reduce(b, op=dist.ReduceOp.SUM)
    ms, e2e_ms_max, _ = t.tolist()
    total_bytes = b[0].item() if not seq_split else qbytes_model(w) * K
    e2e_total = b[1].item()
    if rank != 0:
        return None
    gbs = total_bytes / (ms * 1e-3) / 1e9
    peak, peak_src = peak_hbm()
    # steady state: one step = the attention grid + its combine grid, back to
    # back (programmatic dependent launch overlaps each with its predecessor)
    per_launch_bytes = bytes_total / K
    step_ms = ms / K
    achieved = per_launch_bytes / (step_ms * 1e-3) / 1e9
    kern_avg_ms = kern_ms / max(launches, 1)
    iso = per_launch_bytes / (kern_avg_ms * 1e-3) / 1e9 if launches else None
    kern_name = ("bdk::decode_fast_kernel (stream-K attention over packed blocks + residual) + "
                 "bdk::combine_fast_kernel (LSE merge, commit, fused flush)" if mode == "fast" else
                 "bdk::decode_kernel + combine (bit-faithful dequant, hi/lo split PV)")
    res = {
        "metric": METRIC, "value": round(gbs, 1), "unit": "GB/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": round(ms / K, 5), "latency_us": round(ms / K * 1e3, 2),
        "higher_is_better": True,
        "scaling": "strong" if kind in ("seq", "head") else "weak", "vs_baseline": None,
        "dtype": f"u{w['bits']} codes -> fp16 MMA, fp32 accumulate ({mode} mode)",
        "data": "synthetic (torch.randn fp16 KV; parity pass on the reference's GaussianSource bytes)",
        "mode": mode,
        "config": workload_config(name, world),
        "l2_policy": (f"rotating {n_rep} cache replicas x {per_rep/1e6:.1f} MB quantized per GPU "
                      f"(> 2x L2 {l2/2**20:.0f} MiB); inputs larger than L2, no flush"),
        "exchange": exchange,
        "roofline": {"bound": "hbm",
                     "achieved": round(achieved, 1) if achieved else None,
                     "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4) if achieved else None,
                     "peak_source": peak_src, "kernel": kern_name,
                     "duration": "timed region / steps (each step = attention grid + combine "
                                 "grid, back to back with programmatic dependent launch)",
                     "kernel_avg_us": round(step_ms * 1e3, 2),
                     "kernel_isolated_us": round(kern_avg_ms * 1e3, 2),
                     "isolated_achieved": round(iso, 1) if iso else None,
                     "isolated_note": "CUDA events around each step's launches (no PDL "
                                      "overlap, includes launch latency)",
                     "algorithmic_bytes_per_launch": round(per_launch_bytes),
                     "traffic": load_traffic(name if mode == "fast" else f"{name}_precise")},
        "e2e": ({"value": round(e2e_total / (e2e_ms_max * 1e-3) / 1e9, 2), "unit": "GB/s",
                 "latency_us": round(e2e_ms_max / e2e_steps * 1e3, 1),
                 "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                 "path": ("per rank: pinned host fp16 q (k/v on the last rank) -> H2D -> "
                          "bitkv.decode_partial -> peer/NCCL merge -> D2H fp32 out -> sync"
                          if seq_split else
                          "bitkv.decode_step(host fp32 arrays) -> bdk_decode_step_host (host F16C "
                          "convert to pinned fp16, H2D, decode, fp32 output to pinned host memory "
                          "-- kernel stores when <= 256 KiB, else one D2H copy -- sync, copy out)"),
                 "clock": "host perf_counter (synchronous call), max over ranks"}
                if e2e_ms else None),
        "gpu_launches": n_launched,
        "clocks": clk,
        "prefill_ms_per_replica": round(statistics.median(t_pref), 3),
    }
    return res


# ------------------------------------------------ C4: quantize-and-pack
def run_qpack(args, name, world, rank, local, steps, warmup, soak, sample_clocks=False):
    """Prefill (KVCache::prefill, kvcache.cpp:155-168) of every cell: one
    fused quantize+pack launch per step into a fresh cache."""
    import torch
    import torch.distributed as dist
    from paper_2503_18773_b200 import bitkv as bk

    w = WORKLOADS[name]
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    spec = bk.QuantSpec(w["bits"], bk.QuantAxis.KChannel, w["g"])
    gen = torch.Generator(device=dev)
    gen.manual_seed(4321 + rank)
    shape = (w["batch"], w["hkv"], w["seq"], D)
    k = torch.randn(shape, generator=gen, device=dev, dtype=torch.float16)
    v = torch.randn(shape, generator=gen, device=dev, dtype=torch.float16)
    K, W = steps, warmup
    n_c = min(K, 32)
    caches = [bk.KVCache(w["batch"], w["hkv"], D, w["warp_n"], spec, max_tokens=w["seq"],
                         device=local) for _ in range(n_c)]
    for i in range(W):
        caches[i % n_c].reset()
        caches[i % n_c].prefill_all(k, v)
    torch.cuda.synchronize()
    clocks = Clocks(local) if sample_clocks else None
    if clocks:
        clocks.start()
    t_end = time.time() + soak  # untimed: keeps clocks up while nvidia-smi samples
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
    clk = clocks.stop() if clocks else None
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
    kh, vh = k.cpu().pin_memory(), v.cpu().pin_memory()
    kd, vd = torch.empty_like(k), torch.empty_like(v)
    e2e_steps = 3
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
    per_step = rd + wr
    gbs = per_step * world * K / (ms * 1e-3) / 1e9
    achieved = per_step / (ms / K * 1e-3) / 1e9
    peak, peak_src = peak_hbm()
    return {
        "metric": QPACK_METRIC, "value": round(gbs, 1), "unit": "GB/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": round(ms / K, 5),
        "latency_us": round(ms / K * 1e3, 2), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": f"fp16 -> u{w['bits']} codes (bit-exact integer pack)",
        "data": "synthetic", "config": workload_config(name, world),
        "l2_policy": "inputs 2 x %.0f MB fp16 (> L2), fresh cache per step" % (rd / 2e6),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "peak_source": peak_src,
                     "kernel": "bdk::qpack_fast_kernel (fused quantize + pack, bdk_qpack_fast.cuh)",
                     "duration": "timed region / prefill launches (events, one launch per step)",
                     "algorithmic_bytes_per_launch": per_step,
                     "traffic": load_traffic(name)},
        "e2e": {"value": round(per_step * e2e_steps / e2e_s / 1e9, 2), "unit": "GB/s",
                "latency_us": round(e2e_s / e2e_steps * 1e6, 1),
                "h2d_bytes_per_step": rd, "d2h_bytes_per_step": 0,
                "path": "pinned host fp16 K/V -> H2D -> KVCache.prefill_all (qpack) -> sync",
                "clock": "host perf_counter"},
        "gpu_launches": n_launched, "clocks": clk,
    }


# ------------------------------------------- parity on the reference's bytes
def _errors(got, ref, rows_d):
    import numpy as np
    a = got.astype(np.float64).reshape(-1, rows_d)
    r = ref.astype(np.float64).reshape(-1, rows_d)
    diff = a - r
    nr = np.linalg.norm(r)
    row_rel = np.linalg.norm(diff, axis=1) / np.maximum(np.linalg.norm(r, axis=1), 1e-300)
    return {"max_abs": float(np.abs(diff).max()),
            "rel_l2": float(np.linalg.norm(diff) / nr) if nr > 0 else float(np.linalg.norm(diff)),
            "rel_l2_row_max": float(row_rel.max())}


def parity_decode(name, world, rank, local, steps=3, modes=("fast", "precise"), threads=None,
                  time_ref=False):
    """The GPU decode on run_bench's own bytes vs the reference's decode_step.

    Rank 0 draws the GaussianSource(seed 0) stream in run_bench's order --
    every cell's K [seq*d] then V [seq*d] (b-major, h-minor), then per step q
    [b][hq][d] and per (b, h) k_new[d], v_new[d] (bench.cpp:116-155) -- feeds
    it to the unmodified reference engine (oracle/_ref) and broadcasts it to
    the other ranks, which prefill their share (block range for the sequence
    split).  The reference's outputs are computed before any GPU step so no
    rank waits on the host inside a merge.  Returns (parity dict, reference
    ms per decode step) on rank 0."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_2503_18773_b200 import bitkv as bk
    from paper_2503_18773_b200 import sharding

    w = WORKLOADS[name]
    kind = split_kind(name, world)
    if kind not in ("single", "seq"):
        return None, None
    dev = torch.device("cuda", local)
    threads = threads or os.cpu_count() or 1
    os.environ["BITKV_THREADS"] = str(threads)
    n_r = n_r_of(w)
    B, HQ, HKV, S = w["batch"], w["hq"], w["hkv"], w["seq"]
    if kind == "seq":
        blk_lo, blk_hi = sharding.block_range(S // n_r, world, rank)
        t_lo, t_hi = blk_lo * n_r, (blk_hi * n_r if rank < world - 1 else S)
    else:
        t_lo, t_hi = 0, S
    last = rank == world - 1
    spec = bk.QuantSpec(w["bits"], bk.QuantAxis.KChannel, w["g"])
    caches = {m: bk.KVCache(B, HKV, D, w["warp_n"], spec, max_tokens=(t_hi - t_lo) + steps + n_r,
                            device=local, precise=(m == "precise")) for m in modes}
    cfg = bk.AttentionConfig(batch=B, heads_q=HQ, heads_kv=HKV, head_dim=D,
                             tile_m=max(1, HQ // HKV), tile_n=64, num_splits=4,
                             warp_n=w["warp_n"])
    rc = g = None
    if rank == 0:
        g = O.Gauss(0)
        rc = O.RefCache(B, HKV, D, w["warp_n"], w["bits"], 0, w["g"], True)
    buf = torch.empty((2, S, D), dtype=torch.float16, device=dev)
    for b in range(B):
        for h in range(HKV):
            if rank == 0:
                kv = g.rounded(2 * S * D, threads=threads).reshape(2, S, D)
                rc.prefill(b, h, kv[0], kv[1])
                buf.copy_(torch.from_numpy(kv).to(dev, non_blocking=False).half())
            if world > 1:
                dist.broadcast(buf, 0)
            for c in caches.values():
                c.prefill(b, h, buf[0, t_lo:t_hi], buf[1, t_lo:t_hi])
    # the reference's steps first (host), then the GPU's
    inputs, refs, ref_ms = [], [], []
    for _ in range(steps):
        if rank == 0:
            q = np.zeros((B, HQ, D), np.float32)
            kn = np.zeros((B, HKV, D), np.float32)
            vn = np.zeros((B, HKV, D), np.float32)
            for b in range(B):
                q[b] = g.rounded(HQ * D).reshape(HQ, D)
                for h in range(HKV):
                    kn[b, h] = g.rounded(D)
                    vn[b, h] = g.rounded(D)
            t0 = time.perf_counter()
            refs.append(rc.decode_step(q, kn, vn, tile_n=64, num_splits=4))
            ref_ms.append((time.perf_counter() - t0) * 1e3)
            x = torch.from_numpy(np.concatenate([q.ravel(), kn.ravel(), vn.ravel()])).to(dev)
        else:
            x = torch.empty(B * (HQ + 2 * HKV) * D, dtype=torch.float32, device=dev)
        if world > 1:
            dist.broadcast(x, 0)
        nq = B * HQ * D
        inputs.append((x[:nq].view(B, HQ, D).half(),
                       x[nq:nq + B * HKV * D].view(B, HKV, D).half(),
                       x[nq + B * HKV * D:].view(B, HKV, D).half()))
    rc = None
    errs = {m: None for m in modes}
    comm = sharding.SeqSplitComm(world, B * HQ, D, dev) if kind == "seq" else None
    out = torch.empty((B, HQ, D), dtype=torch.float32, device=dev)
    for m, c in caches.items():
        worst = {"max_abs": 0.0, "rel_l2": 0.0, "rel_l2_row_max": 0.0}
        for s, (q, kn, vn) in enumerate(inputs):
            if kind == "seq":
                bk.decode_partial(c, cfg, q, kn if last else None, vn if last else None, 0,
                                  1 << 30, out=comm.o.view(B, HQ, D), lse=comm.lse.view(B, HQ))
                comm.merge(out)
            else:
                bk.decode_step(c, cfg, q, kn, vn, out=out)
            if rank == 0:
                e = _errors(out.cpu().numpy(), refs[s], D)
                worst = {k: max(worst[k], e[k]) for k in worst}
        if rank == 0:
            tol = TOL[m]
            ok = all(worst[k] < tol[k] for k in tol)
            errs[m] = {**{k: float(f"{v:.3e}") for k, v in worst.items()}, "tol": tol, "pass": ok}
    torch.cuda.synchronize()
    if rank != 0:
        return None, None
    p = {**errs, "steps": steps,
         "source": "run_bench GaussianSource(seed 0) bytes (bench.cpp:18-35, :116-155) -> "
                   "reference decode_step (attention.cpp:164-242, oracle/_ref) vs the GPU path",
         "n_gpus": world}
    return p, (sum(ref_ms[1:]) / max(1, len(ref_ms) - 1) if len(ref_ms) > 1 else ref_ms[0])


def parity_qpack(name, local, threads=None):
    """Bit-exact C4: the GPU prefill of the reference-hashed stream
    (tests/golden/make_golden.py BLOCK_CASES c4_flush_*: GaussianSource(seed),
    per cell K then V) -- sha256 of every packed block of every cell against
    the hashes the reference produced."""
    import numpy as np
    import torch
    from oracle import oracle as O
    from paper_2503_18773_b200 import bitkv as bk

    with open(os.path.join(ROOT, "tests", "golden", "blocks.json")) as f:
        fx = {c["name"]: c for c in json.load(f)}[C4_GOLDEN[name]]
    threads = threads or os.cpu_count() or 1
    spec = bk.QuantSpec(fx["bits"], bk.QuantAxis(fx["k_axis"]), fx["group_size"])
    c = bk.KVCache(fx["batch"], fx["heads_kv"], fx["head_dim"], fx["warp_n"], spec,
                   max_tokens=fx["seq"], device=local)
    g = O.Gauss(fx["seed"])
    S, d = fx["seq"], fx["head_dim"]
    kv = torch.empty((fx["batch"], fx["heads_kv"], 2, S, d), dtype=torch.float16)
    for b in range(fx["batch"]):
        for h in range(fx["heads_kv"]):
            kv[b, h] = torch.from_numpy(g.rounded(2 * S * d, threads=threads).reshape(2, S, d))
    kvd = kv.to(f"cuda:{local}")
    c.prefill_all(kvd[:, :, 0].contiguous(), kvd[:, :, 1].contiguous())  # the timed kernel
    bad = 0
    for cell in fx["cells"]:
        b, h = cell["b"], cell["h"]
        hs = hashlib.sha256()
        for i in range(c.packed_len(b, h) // c.n_r()):
            blk = c.block(b, h, i)
            for a in (blk.k_words, blk.v_words, blk.k_params, blk.v_params):
                hs.update(np.ascontiguousarray(a).astype("<u2").tobytes())
        bad += int(hs.hexdigest() != cell["blocks_sha256"] or
                   c.packed_len(b, h) != cell["packed_len"])
    return {"blocks_bit_exact": bad == 0, "cells_checked": len(fx["cells"]),
            "cells_mismatched": bad,
            "blocks_per_cell": fx["cells"][0]["packed_len"] // fx["n_r"],
            "source": f"tests/golden/blocks.json {C4_GOLDEN[name]} (reference prefill of "
                      f"GaussianSource(seed {fx['seed']}) bytes, sha256 per cell)"}


# ------------------------------------------------------- CPU reference arm
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
                "reference run_bench prefill_seconds (bench.cpp:132-139), full C4 shape, "
                "1 thread by construction")
    g = O.Gauss(0)
    oc = O.OracleCache(w["batch"], w["hkv"], D, w["warp_n"], w["bits"], 0, w["g"], True,
                       max_tokens=w["seq"])
    ks = [g.rounded(w["seq"] * D).reshape(w["seq"], D) for _ in range(2 * w["hkv"])]
    t0 = time.perf_counter()
    for h in range(w["hkv"]):
        oc.prefill(0, h, ks[2 * h], ks[2 * h + 1])
    sec = time.perf_counter() - t0
    return ((rd + wr) / sec / 1e9, sec, "port",
            "oracle C restatement prefill, full C4 shape, 1 thread")


def cpu_reference(w, steps, warm, batch):
    """The unmodified reference engine (oracle/_ref) via its own run_bench, or
    the C restatement (kind "port") when _ref is absent.  Returns (GB/s, mean
    step ms, kind, cores, sample)."""
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    os.environ["BITKV_THREADS"] = str(cores)
    n_r = n_r_of(w)
    qb = qbytes_model(w, batch=batch)
    if O.have_ref():
        r = O.ref_run_bench(mode=1 if batch > 1 else 0, seq_len=w["seq"], batch=batch,
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
        g = O.Gauss(0)
        oc = O.OracleCache(batch, w["hkv"], D, w["warp_n"], w["bits"], 0, w["g"], True,
                           max_tokens=w["seq"] + steps + warm + n_r)
        for b in range(batch):
            for h in range(w["hkv"]):
                k = g.rounded(w["seq"] * D).reshape(w["seq"], D)
                v = g.rounded(w["seq"] * D).reshape(w["seq"], D)
                oc.prefill(b, h, k, v)
        times = []
        for _ in range(warm + steps):
            q = g.rounded(batch * w["hq"] * D).reshape(batch, w["hq"], D)
            kn = g.rounded(batch * w["hkv"] * D).reshape(batch, w["hkv"], D)
            vn = g.rounded(batch * w["hkv"] * D).reshape(batch, w["hkv"], D)
            t0 = time.perf_counter()
            oc.decode_step(q, kn, vn, threads=cores)
            times.append((time.perf_counter() - t0) * 1e3)
        ms = sum(times[warm:]) / steps
        kind = "port"
        sample = (f"oracle C restatement (oracle/bitkv_oracle.c), full shape, {steps} steps, "
                  f"{cores} threads")
    return qb / (ms * 1e-3) / 1e9, ms, kind, cores, sample


def run_reference_arm(args, name, world, rank):
    if rank != 0:
        return None
    w = WORKLOADS[name]
    cfg = workload_config(name, world)
    if w.get("qpack"):
        gbs, sec, kind, sample = cpu_qpack_reference(w)
        return {"impl": "reference", "metric": QPACK_METRIC, "value": round(gbs, 4),
                "unit": "GB/s", "n_gpus": world, "steps": 1, "warmup": 0,
                "ms_per_step": round(sec * 1e3, 3), "latency_us": round(sec * 1e6, 1),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": f"fp32 -> u{w['bits']} codes (CPU)", "data": "synthetic", "config": cfg,
                "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": 1,
                                 "kind": kind, "sample": sample},
                "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
    batch = cfg["global_batch"]
    # bound the run: a reference step is ~0.5 s (C5) to ~3 s (C3) on 16 cores
    est = {"C1": 0.02, "C2": 0.9, "C2b4": 0.9, "C2w2": 0.9, "C3": 3.0, "C5": 0.45}[name]
    est *= (16 / (os.cpu_count() or 16)) * batch / w["batch"]
    cap = max(2, int(150 / max(est, 1e-3)))
    k_run = min(args.steps, cap)
    warm = min(args.warmup, max(1, cap - k_run))
    gbs, ms, kind, cores, sample = cpu_reference(w, k_run, warm, batch)
    if k_run < args.steps:
        sample += f" (K capped at {k_run} of {args.steps} to bound the run)"
    return {"impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s",
            "n_gpus": world, "steps": k_run, "warmup": warm,
            "ms_per_step": round(ms, 3), "latency_us": round(ms * 1e3, 1),
            "higher_is_better": True,
            "scaling": "strong" if split_kind(name, world) in ("seq", "head") else "weak",
            "vs_baseline": None, "dtype": f"u{w['bits']} codes -> fp32 (CPU)",
            "data": "synthetic (GaussianSource seed 0)", "config": cfg,
            "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": cores,
                             "kind": kind, "sample": sample},
            "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


# ------------------------------------------------------------------- main
def condensed(r):
    """The fields of an extra workload's line kept in the headline's extras."""
    if r is None:
        return None
    keep = {k: r[k] for k in ("value", "unit", "latency_us", "n_gpus", "scaling") if k in r}
    keep["workload"] = r["config"]["workload"]
    keep["parallelism"] = r["config"]["parallelism"]
    if "mode" in r:
        keep["mode"] = r["mode"]
    rf = r["roofline"]
    keep["roofline"] = {k: rf.get(k) for k in ("achieved", "peak", "frac", "kernel_isolated_us",
                                               "algorithmic_bytes_per_launch", "traffic")}
    if r.get("e2e"):
        keep["e2e"] = {k: r["e2e"][k] for k in ("value", "unit", "latency_us",
                                                "h2d_bytes_per_step", "d2h_bytes_per_step")}
    keep["gpu_launches"] = r.get("gpu_launches")
    return keep


def dry_run(world, rank):
    """--dry-run: the multi-rank plumbing on CPU (gloo), no CUDA."""
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.tensor([float(rank)])
    ranks = [torch.zeros(1) for _ in range(world)]
    if world > 1:
        dist.all_gather(ranks, t)
        dist.barrier()
    else:
        ranks = [t]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world,
                          "ranks": [int(x.item()) for x in ranks],
                          "config": workload_config(DEFAULT_WORKLOAD, world)}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="fast", choices=["fast", "precise"],
                    help="decode numerics of the headline workload")
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--soak", type=float, default=1.0, help="untimed seconds before timing")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="C5 sequence split: peer-memory merge kernel or NCCL all-gather")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="headline only (no extras, no parity)")
    ap.add_argument("--parity-steps", type=int, default=3)
    ap.add_argument("--dry-run", action="store_true", help="CPU/gloo plumbing check")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.quick:
        args.no_extras = args.no_parity = True
    world, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(self_launch(args.gpus))
    if args.dry_run:
        dry_run(world, rank)
        return
    name = args.workload
    if args.impl == "reference":
        line = run_reference_arm(args, name, world if world > 1 else args.gpus, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    import torch
    import torch.distributed as dist
    if world > 1 and oversubscribed(world):
        local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")
    elif world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        w = WORKLOADS[name]
        if w.get("qpack"):
            res = run_qpack(args, name, world, rank, local, args.steps, args.warmup, args.soak,
                            sample_clocks=True)
        else:
            res = run_decode(args, name, args.mode, world, rank, local, args.steps, args.warmup,
                             args.e2e_steps, args.soak, sample_clocks=True)
        extras = {}
        if not args.no_extras:
            for xn, xm in EXTRAS:
                if xn == name and (xm or "fast") == args.mode:
                    continue
                key = xn + ("_precise" if xm == "precise" else "")
                try:
                    if WORKLOADS[xn].get("qpack"):
                        r = run_qpack(args, xn, world, rank, local, min(args.steps, 50),
                                      args.warmup, 0.2)
                    else:
                        r = run_decode(args, xn, xm, world, rank, local, min(args.steps, 100),
                                       args.warmup, min(args.e2e_steps, 20), 0.2)
                    extras[key] = condensed(r)
                except Exception as e:  # an extra never takes the headline down
                    extras[key] = {"error": f"{type(e).__name__}: {e}"[:300]}
        parity, ref_ms = None, None
        if not args.no_parity:
            par = {}
            par_names = [name] + ([n for n in PARITY if n != name] if not args.no_extras else [])
            for pn in par_names:
                try:
                    if WORKLOADS[pn].get("qpack"):
                        p, rms = (parity_qpack(pn, local) if rank == 0 else None), None
                    else:
                        p, rms = parity_decode(pn, world, rank, local, steps=args.parity_steps)
                except Exception as e:
                    p, rms = {"error": f"{type(e).__name__}: {e}"[:300]}, None
                par[pn] = p
                if pn == name:
                    parity, ref_ms = p, rms
            if rank == 0 and not args.no_extras:
                for qn in ("C4", "C4b2"):
                    if qn != name and qn not in par:
                        try:
                            par[qn] = parity_qpack(qn, local)
                        except Exception as e:
                            par[qn] = {"error": f"{type(e).__name__}: {e}"[:300]}
                for key, x in extras.items():
                    base = key.replace("_precise", "")
                    if x is None or "error" in x or par.get(base) is None:
                        continue
                    p = par[base]
                    if key.endswith("_precise") and "precise" in p:
                        p = {"precise": p["precise"], "steps": p.get("steps")}
                    x["parity"] = p
        if rank == 0:
            res["parity"] = parity
            if extras:
                res["extras"] = extras
            res["cpu_baseline"] = None
            if world == 1 and not args.no_cpu_baseline:
                if w.get("qpack"):
                    gbs, sec, kind, sample = cpu_qpack_reference(w)
                    res["cpu_baseline"] = {"value": round(gbs, 4), "unit": "GB/s", "cores": 1,
                                           "kind": kind, "sample": sample,
                                           "ms_per_step": round(sec * 1e3, 2)}
                elif ref_ms is not None:
                    from oracle import oracle as O
                    qb = qbytes_model(w)
                    res["cpu_baseline"] = {
                        "value": round(qb / (ref_ms * 1e-3) / 1e9, 4), "unit": "GB/s",
                        "cores": os.cpu_count(), "kind": "reference" if O.have_ref() else "port",
                        "ms_per_step": round(ref_ms, 2),
                        "sample": f"reference decode_step (attention.cpp:164-242, oracle/_ref) "
                                  f"on the parity pass's {w['seq']}-token GaussianSource bytes, "
                                  f"{args.parity_steps - 1} timed steps after 1, "
                                  f"BITKV_THREADS={os.cpu_count()}"}
                else:
                    gbs, ms, kind, cores, sample = cpu_reference(w, 2, 1, w["batch"])
                    res["cpu_baseline"] = {"value": round(gbs, 4), "unit": "GB/s",
                                           "cores": cores, "kind": kind, "sample": sample,
                                           "ms_per_step": round(ms, 2)}
            print(json.dumps(res), flush=True)
    finally:
        if world > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
