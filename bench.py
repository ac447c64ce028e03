#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for the B200 2D-Torus all-reduce.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl torus|reference] ...
  (N > 1: launched by torch.distributed.run, one rank per GPU, NCCL process group)

A "step" is one 2D-Torus all-reduce (all SURVEY Sec. 8(a) rows) of the ResNet-50
gradient buffer (25,557,032 elements, synthetic N(0,1)*2^-7 values, per-rank seed
20181113 + rank).  Workloads:
  N >= 2 : fp16 buffer, fp16 wire, mean, grid 2x4 (8), 2x2 (4), 1x2 (2)  -> BASELINE metric
  N == 1 : f32 buffer, fp16 wire, mean: the fused cast/scale-only degenerate case
value = busbw (GB/s) = S * 2(N-1)/N / t, t = max over ranks of the per-call device time
(CUDA events on the launching stream); at N == 1 busbw is 0 by definition and value is
the algbw S/t of the degenerate pass (S = fp16 message bytes).  L2 is flushed (256 MiB
write, then a 256 MiB read that leaves it clean) before every timed call, outside the
events.  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synthetic  # noqa: E402  (seeded inputs only; no method arithmetic)

METRIC = ("2D-torus allreduce busbw GB/s (fp16 25.6M elems, 8×B200, max over ranks) "
          "vs NVLink peak")
NVLINK_NOMINAL = 900.0      # GB/s per direction per GPU (18 x 50)
L2_BYTES = 126 * 1000 * 1000  # B200 L2 (B200_PROFILING.md)
# TORUS_BENCH_OVERSUB=1: run N ranks on fewer GPUs (rank r on GPU r % count, gloo plumbing,
# no NCCL comparator; set TORUS_CTAS to each rank's SM share) to exercise the N = 8 code
# path on a smaller box.  The line is marked "oversubscribed" and is not a measurement.
OVERSUB = os.environ.get("TORUS_BENCH_OVERSUB") == "1"
NVLINK_MEASURED = 770.0     # GB/s per direction, B200_PROFILING.md "peer copy" measurement
DEFAULT_GRID = {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4)}
DT_BYTES = {"f32": 4, "f16": 2, "bf16": 2, "i32": 4}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=400)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--ctas", type=int, default=0, help="CTAs per rank (env TORUS_CTAS)")
    p.add_argument("--impl", default="torus", choices=["torus", "reference"])
    p.add_argument("--grid", default=None, help="XxY (default: 2x4 / 2x2 / 1x2 / 1x1)")
    p.add_argument("--count", type=int, default=synthetic.RESNET50_NUMEL)
    p.add_argument("--dtype", default=None, help="buffer dtype (default f16; f32 at N=1)")
    p.add_argument("--wire", default="f16")
    p.add_argument("--op", default="mean", choices=["sum", "mean"])
    p.add_argument("--algo", default="torus", choices=["torus", "ring", "hier", "nvls"],
                   help="ring / hier = baseline kernels; nvls = in-switch-reduction variant")
    p.add_argument("--no-nccl", action="store_true", help="skip the NCCL comparison")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--e2e-piece", type=int, default=4 << 20,
                   help="elements per pipelined piece of the e2e host-buffer call (0 = one piece)")
    p.add_argument("--no-register", action="store_true",
                   help="do not register the buffer (the pull kernel then copies inputs into the slab)")
    p.add_argument("--no-cpu", action="store_true", help="skip the oracle cpu_baseline leg")
    p.add_argument("--l2", default=None, choices=["flush", "rotate"],
                   help="L2 protocol between timed calls (default: rotate at N=1, flush at N>1)")
    p.add_argument("--out", default=None, help="also append the JSON line to this file")
    return p.parse_args()


# ----------------------------------------------------------------------------------------
# distributed plumbing
# ----------------------------------------------------------------------------------------
def dist_setup(n_gpus):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={world}")
    if OVERSUB:  # code-path check only: several ranks per GPU, gloo plumbing, never a result
        local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        if world > 1:
            dist.init_process_group("gloo")
        return rank, world, local
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def device_align(world):
    """Line the GPUs up right before a timed loop.  The host barrier returns at different
    times on different ranks (100-300 us apart), and a collective's first timed call would
    absorb that skew waiting for its slowest peer.  A one-element NCCL all-reduce enqueued
    on the stream releases every GPU together; the timed calls are enqueued behind it."""
    if world > 1:
        import torch
        import torch.distributed as dist
        dist.all_reduce(torch.zeros(1, device="cuda"))
        torch.cuda._sleep(2_000_000)  # ~1 ms on every GPU while the hosts enqueue ahead


def gather_max(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------------------
# clocks (B200_PROFILING.md "clocks DURING the timed region")
# ----------------------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, enabled):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
        if enabled:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            try:
                self.fh = open(self.path, "w")
                self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}",
                                              "--format=csv,noheader,nounits", "-lms", "200"],
                                             stdout=self.fh, stderr=subprocess.DEVNULL)
                # nvidia-smi takes ~0.5-1 s to start on a multi-GPU box: wait for its first
                # sample so the warm-up and the (short) timed region are both covered
                t0 = time.perf_counter()
                while os.path.getsize(self.path) == 0 and time.perf_counter() - t0 < 5.0:
                    time.sleep(0.05)
            except OSError:
                self.proc = None

    def stop(self, n_gpus):
        if not self.proc:
            return None
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9 or not f[0].isdigit() or int(f[0]) >= n_gpus:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        top = sorted(sm)[len(sm) // 2:]  # samples under load: upper half
        return {"sm_mhz": statistics.median(top), "sm_max_mhz": max(mx),
                "samples": len(sm), "reasons": sorted(reasons)}


class NvlinkCounters:
    """NVML NVLink data counters of this rank's GPU (KiB, cumulative, summed over links):
    NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX (user payload, no protocol overhead) and
    _RAW_TX / _RAW_RX (payload + protocol).  Read around a block of calls they give the
    NVLink bytes per call measured by the hardware, without a profiler."""
    FIELDS = {"data_tx": 138, "data_rx": 139, "raw_tx": 140, "raw_rx": 141}

    def __init__(self, local):
        self.h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            bus = None
            import torch
            props = torch.cuda.get_device_properties(local)
            bus = getattr(props, "pci_bus_id", None)
            if bus is not None:
                for i in range(pynvml.nvmlDeviceGetCount()):
                    hh = pynvml.nvmlDeviceGetHandleByIndex(i)
                    if pynvml.nvmlDeviceGetPciInfo(hh).bus == bus:
                        self.h = hh
            if self.h is None:
                vis = os.environ.get("CUDA_VISIBLE_DEVICES")
                idx = int(vis.split(",")[local]) if vis else local
                self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nvml = pynvml
            self.links = 18
        except Exception:  # no NVML: counters unavailable
            self.h = None

    def read(self):
        if self.h is None:
            return None
        out = {}
        any_ok = False
        try:
            for name, fid in self.FIELDS.items():
                vals = self.nvml.nvmlDeviceGetFieldValues(self.h, [(fid, l) for l in range(self.links)])
                tot = 0
                for v in vals:
                    if v.nvmlReturn == 0:
                        tot += int(v.value.ullVal)
                        any_ok = True
                out[name] = tot * 1024  # KiB -> bytes
        except Exception:
            return None
        # NOT_SUPPORTED on every link (e.g. this pool's containers: profiles/r02_nvml_probe.txt)
        return out if any_ok else None

    @staticmethod
    def per_call(a, b, calls):
        if a is None or b is None or calls <= 0:
            return None
        return {k: (b[k] - a[k]) / calls for k in a}


# ----------------------------------------------------------------------------------------
# the torus arm
# ----------------------------------------------------------------------------------------
def make_input(args, rank, dtype_s):
    dist_name = "grad"
    a = synthetic.make(dist_name, args.count, rank, dtype_s if dtype_s != "bf16" else "bf16")
    return a


def to_tensor(a, dtype_s, device):
    import torch
    if dtype_s == "bf16":
        return torch.from_numpy(a.view(np.int16).copy()).view(torch.bfloat16).to(device)
    return torch.from_numpy(a).to(device)


def run_torus(args):
    import torch
    import torch.distributed as dist
    from paper_1811_05233_b200 import TorusComm

    rank, world, local = dist_setup(args.gpus)
    dev = torch.device("cuda", local)
    X, Y = (tuple(int(v) for v in args.grid.lower().split("x")) if args.grid
            else DEFAULT_GRID.get(world, (world, 1)))
    dtype_s = args.dtype or ("f32" if world == 1 else "f16")
    wire_s = args.wire if dtype_s == "f32" else dtype_s
    TD = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16, "i32": torch.int32}
    D = args.count
    S = D * DT_BYTES[wire_s]                    # message bytes on the wire (BASELINE: fp16)
    bus = 2.0 * (world - 1) / world

    comm = TorusComm.init(X=X, Y=Y)
    host = make_input(args, rank, dtype_s)
    x0 = to_tensor(host, dtype_s, dev)
    buf = x0.clone()
    if world > 1 and not args.no_register:
        comm.register(buf)  # zero-copy: peers read this buffer directly (torus_register_buffer)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    clean = torch.zeros(64 << 20, dtype=torch.int32, device=dev)  # 256 MiB, read only

    def evict(s):
        """Untimed L2 eviction between timed calls: write 256 MiB (> 126 MB L2), then read
        another 256 MiB so the flush's dirty lines are written back here, not inside the
        timed call."""
        flush.fill_(s & 0xFF)
        clean.max()

    if args.algo == "nvls":
        comm.nvls_init(D * DT_BYTES[wire_s] + (4 << 20))
    reduce_fn = {"ring": comm.ring_all_reduce, "hier": comm.hier_all_reduce,
                 "nvls": comm.nvls_all_reduce}.get(args.algo, comm.all_reduce)

    def call(b=None):
        reduce_fn(buf if b is None else b, op=args.op, wire=TD[wire_s], stream=stream)

    # L2 protocol between timed calls.  N > 1 (NVLink-bound): evict before every call.  N = 1
    # (HBM-bound): rotate over buffers whose total exceeds 3x L2 with no eviction, so each
    # call reads a cold buffer AND writes back the dirty lines the previous call left in L2
    # -- the steady state of back-to-back kernels.  (An eviction that leaves L2 clean lets
    # ~58 MB of this call's writes be written back after its end event, which puts the
    # algorithmic-byte rate above the HBM peak.)
    l2_mode = args.l2 or ("rotate" if world == 1 else "flush")
    ring = [buf]
    if l2_mode == "rotate":
        nbytes = buf.numel() * buf.element_size()
        ring += [x0.clone() for _ in range(max(2, -(-3 * L2_BYTES // nbytes)) - 1)]

    # sanity (not the parity gate -- that is tests/): all ranks agree, and the result is
    # within the north-star tolerance of an f64 all-reduce done with NCCL in f64.
    buf.copy_(x0)
    call()
    torch.cuda.synchronize()
    sanity = {}
    if world > 1:
        ref = x0.double()
        dist.all_reduce(ref)
        if args.op == "mean":
            ref /= world
        mag = x0.double().abs()
        dist.all_reduce(mag)
        if args.op == "mean":
            mag /= world
        err = float(((buf.double() - ref).abs() / (mag + 1e-30)).max())
        cs = buf.view(torch.uint8).to(torch.int64).sum()
        cs_all = [torch.zeros_like(cs) for _ in range(world)]
        dist.all_gather(cs_all, cs)
        sanity = {"ranks_identical": all(int(c) == int(cs_all[0]) for c in cs_all),
                  "max_err_over_sum_abs_vs_f64": err}
    else:
        ref = x0.to(TD[wire_s]).to(x0.dtype)
        sanity = {"ranks_identical": True, "equals_cast_roundtrip": bool(torch.equal(buf, ref))}
    if comm.async_error():
        raise SystemExit("device watchdog fired")

    # ---- device-timed region (the clock sampler starts before the warm-up) ----
    clocks = Clocks(rank == 0)
    t_w = time.perf_counter()
    while True:  # warm-up: >= W calls and >= 0.5 s so the sampler has seen load
        for i in range(max(args.warmup, 3)):
            call(ring[i % len(ring)])
        torch.cuda.synchronize()
        if gather_max(time.perf_counter() - t_w, world) > 0.5:
            break
    barrier(world)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    torch.cuda.synchronize()
    barrier(world)
    device_align(world)
    if l2_mode == "flush":
        evict(0)
    call(ring[-1])  # untimed: the first call after the idle barrier pays a wake-up (profiles/r02_ab*.txt: call 0)
    for s in range(args.steps):
        if l2_mode == "flush":
            evict(s)                            # L2 evicted and clean, untimed
        ev[s][0].record(stream)
        call(ring[s % len(ring)])
        ev[s][1].record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clk = clocks.stop(args.gpus) if rank == 0 else None
    times = [a.elapsed_time(b) * 1e-3 for a, b in ev]   # seconds
    t_local = sum(times) / len(times)
    t = gather_max(t_local, world)
    t_min = gather_max(min(times), world)
    srt = sorted(times)
    t_p50 = gather_max(srt[len(srt) // 2], world)
    t_p90 = gather_max(srt[min(len(srt) - 1, (9 * len(srt)) // 10)], world)
    t_max = gather_max(srt[-1], world)
    algbw = S / t / 1e9
    busbw = algbw * bus
    if comm.async_error():
        raise SystemExit("device watchdog fired during timing")

    # ---- NVLink bytes per call, measured by the hardware (NVML counters, untimed) ----
    nvl_torus = nvl_nccl = None
    nvl = NvlinkCounters(local) if world > 1 else None
    if nvl is not None and nvl.h is not None:
        torch.cuda.synchronize()
        barrier(world)
        c0 = nvl.read()
        for _ in range(args.steps):
            call()
        torch.cuda.synchronize()
        c1 = nvl.read()
        nvl_torus = gather_counters(NvlinkCounters.per_call(c0, c1, args.steps), world)

    # ---- NCCL comparator on the same tensor (like for like: AVG for mean) ----
    nccl = None
    if world > 1 and not args.no_nccl:
        op = dist.ReduceOp.AVG if args.op == "mean" else dist.ReduceOp.SUM
        for _ in range(max(args.warmup, 3)):
            dist.all_reduce(buf, op=op)
        torch.cuda.synchronize()
        barrier(world)
        evn = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        ns = torch.cuda.current_stream()
        device_align(world)
        evict(0)
        dist.all_reduce(buf, op=op)  # untimed, as for the torus arm
        for s in range(args.steps):
            evict(s)
            evn[s][0].record(ns)
            dist.all_reduce(buf, op=op)
            evn[s][1].record(ns)
        torch.cuda.synchronize()
        tn = gather_max(sum(a.elapsed_time(b) for a, b in evn) * 1e-3 / args.steps, world)
        if nvl is not None and nvl.h is not None:
            torch.cuda.synchronize()
            barrier(world)
            c0 = nvl.read()
            for _ in range(args.steps):
                dist.all_reduce(buf, op=op)
            torch.cuda.synchronize()
            c1 = nvl.read()
            nvl_nccl = gather_counters(NvlinkCounters.per_call(c0, c1, args.steps), world)
        nccl = {"busbw": S / tn / 1e9 * bus, "algbw": S / tn / 1e9, "us": tn * 1e6,
                "nvlink_bytes_per_call": nvl_nccl,
                "version": ".".join(map(str, torch.cuda.nccl.version())),
                "nvls_env": os.environ.get("NCCL_NVLS_ENABLE", "default")}
        buf.copy_(x0)

    # ---- e2e through the public API with HOST buffers: H2D, all-reduce, D2H ----
    e2e = None
    if not args.no_e2e:
        hbuf = (torch.from_numpy(host.view(np.int16).copy()).view(torch.bfloat16) if dtype_s == "bf16"
                else torch.from_numpy(host.copy())).pin_memory()
        piece = args.e2e_piece
        if args.algo == "torus":
            def e2e_step():
                comm.all_reduce_host(hbuf, buf, op=args.op, wire=TD[wire_s], piece=piece, stream=stream)
            how = (f"torus_allreduce_host (C-ABI): pinned host buffer, H2D + all-reduce + D2H "
                   f"pipelined over pieces of {piece} elements on two copy streams")
        else:
            hout = torch.empty_like(hbuf).pin_memory()

            def e2e_step():
                buf.copy_(hbuf, non_blocking=True)
                call()
                hout.copy_(buf, non_blocking=True)
            how = "H2D copy, all-reduce, D2H copy on one stream"
        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        device_align(world)
        e0.record(stream)
        for s in range(args.steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        te = gather_max(e0.elapsed_time(e1) * 1e-3 / args.steps, world)
        nb = host.nbytes
        e2e = {"value": (S / te / 1e9) * (bus if world > 1 else 1.0),
               "unit": "GB/s", "us_per_step": te * 1e6,
               "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb, "how": how}

    if l2_mode == "flush":
        l2_desc = ("flushed before every timed call (256 MiB write, then 256 MiB read so no dirty "
                   "flush lines are written back inside the timed call)")
    else:
        l2_desc = (f"no flush: {len(ring)} buffers of {buf.numel() * buf.element_size()} B in rotation "
                   f"(> 3x the 126 MB L2), so every call reads a cold buffer and pays the write-back "
                   f"of the dirty lines the previous call left in L2")
    launches = comm.launches(D, TD[dtype_s], TD[wire_s])
    # ---- roofline of the dominant (only) kernel ----
    if world > 1:
        kname = kernel_name(comm, D, TD, dtype_s, wire_s)
        tkey = "ll128" if kname == "torus_ll128_kernel" else "torus"
        alg_bytes = bus * S                        # NVLink bytes per rank per call
        achieved = alg_bytes / t / 1e9             # t is per call (all rounds)
        roof = {"bound": "nvlink", "achieved": achieved, "peak": NVLINK_MEASURED,
                "unit": "GB/s", "frac": achieved / NVLINK_MEASURED,
                "frac_of_nominal_900": achieved / NVLINK_NOMINAL,
                "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s/direction "
                               "(MEASURED_PEAKS.json has no NVLink entry)",
                "traffic": load_traffic(f"{tkey}_{X}x{Y}"), "kernel": kname,
                "algorithmic_bytes_per_call": alg_bytes,
                "nvlink_tx_bytes_ncu": load_traffic(f"{tkey}_{X}x{Y}_nvltx"),
                "nvlink_tx_user_bytes_ncu": load_traffic(f"{tkey}_{X}x{Y}_nvltx_user"),
                "traffic_source": "profiles/traffic.json (ncu on rank 0 of a real run, profiles/r02_ncu_*.csv)",
                "nvlink_bytes_per_call_nvml": nvl_torus}
    else:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
            os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
        hbm = peaks.get("hbm_gbs", 6650.0)
        alg_bytes = 2.0 * D * DT_BYTES[dtype_s] if dtype_s != wire_s else 0.0
        achieved = alg_bytes / t / 1e9 if launches else 0.0
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650",
                "traffic": load_traffic(kernel_name(comm, D, TD, dtype_s, wire_s).replace("_kernel", "")),
                "kernel": kernel_name(comm, D, TD, dtype_s, wire_s),
                "algorithmic_bytes_per_call": alg_bytes}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args, X, Y, dtype_s, wire_s, world)

    comm.destroy()
    if rank != 0:
        return
    value = busbw if world > 1 else algbw
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": wire_s, "data": "synthetic",
        "config": {"workload": ("resnet50-grad-allreduce" if world > 1 else
                                "resnet50-grad-castscale-degenerate (N=1)"),
                   "count": D, "buffer_dtype": dtype_s, "wire_dtype": wire_s, "op": args.op,
                   "grid": f"ring{world}" if args.algo == "ring" else f"{X}x{Y}",
                   "algo": args.algo,
                   "parallelism": (f"ring{world}" if args.algo == "ring" else f"{args.algo}{X}x{Y}"),
                   "ctas_per_rank": comm_ctas(),
                   "buffer": ("registered (zero-copy)" if world > 1 and not args.no_register
                              else "unregistered"),
                   "message_bytes": S, "l2": l2_desc,
                   "value_is": "busbw" if world > 1 else "algbw (busbw is 0 at N=1)",
                   **({"oversubscribed": "several ranks per GPU: a code-path check, not a measurement"}
                      if OVERSUB else {})},
        "algbw": algbw, "busbw": busbw, "us_per_call": t * 1e6, "us_per_call_min": t_min * 1e6,
        "us_per_call_p50": t_p50 * 1e6, "us_per_call_p90": t_p90 * 1e6, "us_per_call_max": t_max * 1e6,
        "frac_nvlink_900": busbw / NVLINK_NOMINAL if world > 1 else None,
        "gpu_launches": launches * args.steps,
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "nccl": nccl, "clocks": clk,
        "sanity": sanity,
    }
    emit(line, args)


_CTAS = [None]


def gather_counters(d, world):
    """max over ranks of each NVML counter delta (None if any rank lacks NVML)"""
    if world == 1 or d is None:
        return d
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, d)
    if any(o is None for o in out):
        return None
    return {k: max(o[k] for o in out) for k in d} | {"ranks": out}


def kernel_name(comm, D, TD, dtype_s, wire_s):
    try:
        return comm.route(D, TD[dtype_s], TD[wire_s])
    except Exception:
        return "torus_kernel"


def comm_ctas():
    return _CTAS[0]


def load_traffic(kernel):
    """dram bytes per launch from a committed ncu --set full capture, if present."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        v = json.load(open(p)).get(kernel)
        return float(v) if v is not None else None
    except (OSError, ValueError, TypeError):
        return None


def emit(line, args):
    s = json.dumps(line)
    print(s, flush=True)
    if args.out:
        with open(args.out, "a") as f:
            f.write(s + "\n")


# ----------------------------------------------------------------------------------------
# the oracle (CPU) legs: cpu_baseline and --impl reference
# ----------------------------------------------------------------------------------------
def oracle_sample_size(X, Y, steps=1):
    # bounded single-threaded oracle work: ~0.1-0.3 s per step (1M elements at 2x4),
    # smaller samples for long --steps runs so the reference arm ends within minutes
    base = (1 << 22) if X * Y == 1 else (1 << 20)
    return base if steps <= 200 else base // 4


_ORACLE_INPUTS = {}


def time_oracle(X, Y, dtype_s, wire_s, op, D):
    import oracle
    N = X * Y
    key = (D, N, dtype_s)
    if key not in _ORACLE_INPUTS:  # generated once; the oracle reads them, never writes
        _ORACLE_INPUTS.clear()
        _ORACLE_INPUTS[key] = synthetic.make_all("grad", D, N, dtype_s)
    ins = _ORACLE_INPUTS[key]
    oracle.lib()
    t0 = time.perf_counter()
    oracle.torus_allreduce(ins, X, Y, dtype_s, wire=wire_s, op=op, q=16 // DT_BYTES[wire_s])
    return time.perf_counter() - t0


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(args, X, Y, dtype_s, wire_s, world):
    D = min(args.count, oracle_sample_size(X, Y))
    reps, tot = 0, 0.0
    # single-threaded oracle pinned to one core (SURVEY 8(d) "oracle timing beside it")
    old_aff = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
    core = min(old_aff) if old_aff else None
    if core is not None:
        os.sched_setaffinity(0, {core})
    try:
        while tot < 10.0 and reps < 50:
            tot += time_oracle(X, Y, dtype_s, wire_s, args.op, D)
            reps += 1
    finally:
        if old_aff:
            os.sched_setaffinity(0, old_aff)
    t = tot / reps
    S = D * DT_BYTES[wire_s]
    bus = 2.0 * (world - 1) / world
    v = S / t / 1e9 * (bus if world > 1 else 1.0)
    return {"value": v, "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": f"{X}x{Y} grid, {D} of {args.count} elements, {dtype_s} buffer / "
                      f"{wire_s} wire, {args.op}; {reps} reps, {t:.3f} s each, "
                      f"single-threaded C (oracle/torus_oracle.c), pinned to core {core}",
            "host_cpus": os.cpu_count(), "cpu_model": cpu_model()}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    X, Y = (tuple(int(v) for v in args.grid.lower().split("x")) if args.grid
            else DEFAULT_GRID.get(world, (world, 1)))
    dtype_s = args.dtype or ("f32" if world == 1 else "f16")
    wire_s = args.wire if dtype_s == "f32" else dtype_s
    # the full workload when (steps + warm-up) oracle runs fit in ~3 minutes of one core
    # (~0.8 s per simulated rank for 25.6M elements), else a bounded sample
    full = (args.steps + max(args.warmup, 1)) * X * Y * 0.8 * args.count / 25_557_032 <= 200.0
    D = args.count if full else min(args.count, oracle_sample_size(X, Y, args.steps))
    for _ in range(max(args.warmup, 1)):
        time_oracle(X, Y, dtype_s, wire_s, args.op, D)
    ts = [time_oracle(X, Y, dtype_s, wire_s, args.op, D) for _ in range(args.steps)]
    t = sum(ts) / len(ts)
    S = D * DT_BYTES[wire_s]
    bus = 2.0 * (world - 1) / world
    v = S / t / 1e9 * (bus if world > 1 else 1.0)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": wire_s,
        "data": "synthetic",
        "config": {"workload": ("resnet50-grad-allreduce" if world > 1 else
                                "resnet50-grad-castscale-degenerate (N=1)"),
                   "count": args.count, "buffer_dtype": dtype_s, "wire_dtype": wire_s,
                   "op": args.op, "grid": f"{X}x{Y}", "parallelism": f"torus{X}x{Y}"},
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": (f"the full workload: {D} elements per rank per step" if D == args.count
                                    else f"{D} of {args.count} elements per rank per step")
                                   + f", {X}x{Y} simulated ranks, single-threaded C oracle",
                         "cpu_model": cpu_model()},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    emit(line, args)


def main():
    args = parse()
    if args.ctas:
        os.environ["TORUS_CTAS"] = str(args.ctas)
    if OVERSUB:
        args.no_nccl = True
    if args.impl == "reference":
        run_reference(args)
        return
    import paper_1811_05233_b200.torus as T
    orig_init = T.TorusComm.init

    def init_and_record(*a, **k):
        c = orig_init(*a, **k)
        _CTAS[0] = c.ctas()
        return c
    T.TorusComm.init = init_and_record
    run_torus(args)
    try:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()
    except Exception:
        pass


if __name__ == "__main__":
    main()
