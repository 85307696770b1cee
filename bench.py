#!/usr/bin/env python3
"""bench.py — B200 loop-nest execution backend benchmark (one JSON line).

Workload (every N): BASELINE.json configs[4], the seismic wave4 4th-order 3-D
acoustic wave propagation nest, 1024^3 fp32, in the saturated form, one time
step per step (3-level buffer rotation up <- u <- un), strong-scaled over N
z slabs (the scaling case of the metric's "1/2/4/8 GPU").
N = 1 runs the same slab code with one slab (no neighbours = a plain launch),
so BENCH N=1 and SCALE N=1 are the same measurement.  `per_kernel` covers
every BASELINE nest (configs[0]-[3] and zsolve) in the original and
saturated forms; `--workload d3q19` runs configs[1] (D3Q19 256^3 fp64,
weak-scaled z slabs for N > 1) as the headline instead.

  value   algorithmic GB/s of the step with inputs resident in HBM (16 B per
          point for wave4: 3 reads + 1 write of 4 B), whole
          job over all ranks (max-over-ranks step time).  Inputs (17 GB) are
          far larger than the 126 MB L2: no flush needed between steps.
  e2e     the same metric through the public host-buffer API: pinned
          reference-layout host arrays -> H2D -> remap -> kernel -> remap ->
          D2H, every copy inside the timed region.

--impl reference: the reference's own CPU path for the nest — the reference
optimizer's emitted accsat C compiled by gcc -O3 -ffp-contract=off (satcc's
wrapper mode, proj/tools/satcc_main.cpp:285-360), OpenMP over all host
cores, inputs generated on the host (oracle/fill.c), nothing from this
repo's GPU library loaded.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

METRIC = "per-kernel GB/s (% B200 HBM roofline), saturated vs original speedup, 1/2/4/8 GPU"

WORKLOADS = {
    # name: (kernel id(s), dtype, grid per --size default, scaling)
    "wave4": ("wave4.c:wave4:0", "f32", 1024, "strong"),
    "d3q19": ("d3q19.c:stream_collide:0", "f64", 256, "weak"),
    # multi-kernel time steps of the 2-D nests (BASELINE configs[2], configs[3])
    "swim": (["swim.c:calc1:0", "swim.c:calc2:1", "swim.c:calc3:2"], "f64", 8192, "strong"),
    "clover": (["clover.c:ideal_gas:0", "clover.c:pdv_predict:1", "clover.c:advec_cell_x:2"], "f64", 7680, "strong"),
}

# per-kernel table: (kernel id, BASELINE size, dtype, sweeps per step)
TABLE = [
    ("jacobi7.c:jacobi7:0", 256, "f64", 100),
    ("d3q19.c:stream_collide:0", 256, "f64", 1),
    ("swim.c:calc1:0", 8192, "f64", 1),
    ("swim.c:calc2:1", 8192, "f64", 1),
    ("swim.c:calc3:2", 8192, "f64", 1),
    ("clover.c:ideal_gas:0", 7680, "f64", 1),
    ("clover.c:pdv_predict:1", 7680, "f64", 1),
    ("clover.c:advec_cell_x:2", 7680, "f64", 1),
    ("wave4.c:wave4:0", 1024, "f32", 1),
    ("zsolve.c:z_solve_lhs:0", 256, "f64", 1),
]

REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [s[0] for s in self.samples]
        mask = 0
        for s in self.samples:
            mask |= s[2]
        reasons = [n for b, n in REASON_BITS.items() if mask & b and n != "gpu_idle"]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(self.samples)}


def workload_config(workload, size, ws, variant):
    """The `config` object — identical in both arms (ours and --impl reference)."""
    kid, dtype, _, scaling = WORKLOADS[workload]
    if workload == "wave4":
        grid = [size] * 3
        name = ("seismic wave4 4th-order 3-D acoustic wave propagation fp32 (BASELINE configs[4]), "
                "one time step per step, 3-level buffer rotation")
        bpp = 16
    elif workload == "swim":
        grid = [size] * 2
        name = "swim shallow-water time step calc1 -> calc2 -> calc3 fp64 (BASELINE configs[2])"
        bpp = 56 + 80 + 120
    elif workload == "clover":
        grid = [size] * 2
        name = "CloverLeaf-style hydro step ideal_gas -> PdV -> advec_cell_x fp64 (BASELINE configs[3])"
        bpp = 32 + 96 + 48
    else:
        grid = [size, size, size * ws]
        name = ("D3Q19 lattice-Boltzmann collide+stream (olbm-like) fp64 (BASELINE configs[1]), "
                "one sweep per step, src <-> dst")
        bpp = 305
    return {"workload": name, "kernel_id": kid, "grid": grid, "form": variant, "dtype": dtype,
            "bytes_per_point": bpp, "points": int(np.prod(grid)), "scaling": scaling,
            "l2": "inputs >> 126 MB L2 (no flush needed)"}


def dist_setup(args):
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        if os.environ.get("ACS_BENCH_SAME_DEVICE"):
            # functional check of the N-rank path on a one-GPU box (numbers meaningless)
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
            return rank, ws, 0, dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return rank, ws, local, dist
    if torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, ws, local, None


def time_steps(fn, steps, warmup, stream, dist=None):
    """W untimed steps, then K steps between CUDA events on `stream`,
    synchronize + barrier on both sides; returns max-over-ranks ms/step."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    return ms


def time_reps(fn, reps, warmup, stream):
    """Per-repetition CUDA-event times (ms) of `fn` on `stream`."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record(stream)
    for i in range(reps):
        fn()
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    return [ev[i].elapsed_time(ev[i + 1]) for i in range(reps)]


def stats(ms):
    q1, med, q3 = (float(x) for x in np.percentile(ms, [25, 50, 75]))
    return med, q3 - q1


# ---------------------------------------------------------------------------
# the headline: slab-sharded time steps (N = 1: one slab)

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="wave4", choices=sorted(WORKLOADS))
    ap.add_argument("--variant", default="accsat")
    ap.add_argument("--schedule", default="default")
    ap.add_argument("--size", type=int, default=0, help="interior extent (default: the BASELINE size)")
    ap.add_argument("--no-table", action="store_true", help="skip the per-kernel table")
    ap.add_argument("--table-reps", type=int, default=30)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="enqueue every step eagerly (no CUDA graph)")
    ap.add_argument("--exchange", default="auto", choices=["auto", "peer", "nccl"],
                    help="N>1 halo path: peer memory (CUDA IPC write-through), NCCL P2P, or auto (peer, else NCCL)")
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--e2e-chunks", type=int, default=16)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    args.size = args.size or WORKLOADS[args.workload][2]
    if isinstance(args.schedule, str) and args.schedule.isdigit():
        args.schedule = int(args.schedule)     # an explicit registered slot (0 = naive)

    if args.impl == "reference":
        return reference_arm(args)

    import torch
    from paper_2306_13002_b200 import shard
    rank, ws, local, dist = dist_setup(args)
    peak, peak_kind = load_peaks()
    kid, dtype, _, scaling = WORKLOADS[args.workload]
    size = {"wave4": (args.size,) * 3, "d3q19": (args.size * ws, args.size, args.size)}.get(
        args.workload, (args.size, args.size))
    sr = shard.SlabRank(kid, size, ws, rank, dtype=dtype, variant=args.variant, schedule=args.schedule)
    stream = torch.cuda.current_stream()
    tuned = None
    if args.schedule == "default" and args.variant != "original":
        tuned = []
        for k, lw in zip(sr.ks, sr.ws):                                  # untimed autotune, per kernel
            names = [a.name for a in lw.spec.arrays]
            tuned.append(k.tune({n: sr.buf[n] for n in names}, dict(lw.scalars), args.variant, reps=15)[0])
        sr.schedule = tuned if sr.multi else tuned[0]
        sr.refill()
    torch.cuda.synchronize()
    exchange = "none"
    if ws > 1:
        exchange = connect_ranks(args, sr, dist, rank, ws)
        if exchange is None:
            return 3
    graph = False
    if sr.mode != "p2p" and not args.no_graph:
        sr.capture(stream)
        graph = True
    if dist:
        dist.barrier()
    per_step = sr.launches_per_step()
    for _ in range(args.warmup):
        sr.step(stream=stream)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms = time_steps(lambda: sr.step(stream=stream), args.steps, 0, stream, dist)
    local_bytes = sr.algorithmic_bytes
    total_bytes = sr.global_bytes
    value = total_bytes / (ms * 1e-3) / 1e9
    scheds = sr.schedule if isinstance(sr.schedule, list) else [sr.schedule]
    sched_name = "; ".join(k.info["schedules"][1 if dtype == "f32" else 0][sc] if isinstance(sc, int) else str(sc)
                           for k, sc in zip(sr.ks, scheds))
    out = {"metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": scaling,
           "vs_baseline": None, "dtype": dtype,
           "data": "synthetic (seeded SplitMix64, SURVEY.md §8d distributions; generated in HBM)",
           "config": workload_config(args.workload, args.size, ws, args.variant),
           "gpu_launches": per_step * args.steps,
           "execution": {"parallelism": f"z-slab sharding x{ws}" + ("" if ws == 1 else f", exchange: {exchange}"),
                         "slab_planes": sr.plan.owned(rank)[1] - sr.plan.owned(rank)[0],
                         "step": ("one CUDA graph replay per step: " +
                                  ("wait_ctr -> sharded launch (write-through) -> signal_ctr" if sr.mode == "peer"
                                   else "one launch")) if graph else
                                 ("boundary planes -> NCCL P2P halo exchange on a comm stream | interior planes"
                                  if sr.mode == "p2p" else "eager launch"),
                         "schedule": sched_name, "tuned_slot": tuned,
                         "layout": "row-major, 16-element padded pitch, sector-aligned rows"
                                   if args.workload == "wave4" else "q-major SoA"}}
    achieved = local_bytes / (ms * 1e-3) / 1e9
    kname = {"wave4": "wave4_f32", "d3q19": "stream_collide", "swim": "calc1+calc2+calc3",
             "clover": "ideal_gas+pdv_predict+advec_cell_x"}[args.workload]
    out["roofline"] = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                       "frac": round(achieved / peak, 4), "peak_kind": peak_kind,
                       "traffic": load_traffic(kname),
                       "kernel": f"{kname} {args.variant}: {sched_name}",
                       "per_unit": f"{sum(lw.bytes_per_point for lw in sr.ws)} B/point x {sr.w.points} points "
                                   "per step (rank 0's slab), over the step's CUDA-event time"}
    out["clocks"] = clk.summary()
    if not args.no_e2e:
        if ws == 1 and not sr.multi:
            sr.close()
            del sr.buf
            torch.cuda.empty_cache()
            out["e2e"] = e2e_host_runner(args, sr.gw, sr.k, dist)
        else:
            out["e2e"] = e2e_sharded(args, sr, dist, ws)
    sr.close()
    del sr
    torch.cuda.empty_cache()
    if not args.no_table and ws == 1:
        out["per_kernel"] = per_kernel_table(peak, args.table_reps)
    if rank == 0 and ws == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(args)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out))
    return 0


def connect_ranks(args, sr, dist, rank, ws):
    """Wires the slab neighbours: CUDA-IPC peer memory (write-through from the
    kernel), else NCCL P2P halo exchange.  Never falls back to replicas:
    returns None (the bench then exits non-zero) when neither works."""
    err = None
    if args.exchange in ("auto", "peer"):
        exp = [None] * ws
        dist.all_gather_object(exp, sr.export())
        try:
            sr.connect_ipc(exp[rank - 1] if rank > 0 else None, exp[rank + 1] if rank < ws - 1 else None)
        except Exception as e:     # no peer access between these GPUs
            err = str(e)[:200]
        errs = [None] * ws
        dist.all_gather_object(errs, err)
        err = next((e for e in errs if e), None)
        if err is None:
            return "peer memory (CUDA IPC over NVLink), in-kernel write-through + device flags"
        sr.close()
        sr.lo_ptr, sr.hi_ptr, sr.lo_flag, sr.hi_flag = {}, {}, None, None
        print(f"[bench] rank {rank}: peer memory unavailable ({err})", file=sys.stderr)
        if args.exchange == "peer":
            return None
    try:
        sr.connect_p2p(dist)
    except NotImplementedError as e:
        print(f"[bench] rank {rank}: {e}", file=sys.stderr)
        return None
    return "NCCL P2P (torch.distributed batch_isend_irecv) overlapped with interior planes" + \
        (f"; peer memory unavailable: {err}" if err else "")


def e2e_sharded(args, sr, dist, ws):
    """Per rank per step: the owned planes of every input array from pinned
    reference-layout host memory -> device staging -> native remap, queued
    AFTER the step's wait for the neighbours (their write-through into this
    rank's halos / push targets cannot race the upload); the sharded step;
    the owned planes of the produced array -> staging -> D2H."""
    import torch
    from paper_2306_13002_b200 import backend, nests
    stream = torch.cuda.current_stream()
    names = sr.names
    lo, hi = sr.plan.local_range(sr.rank)
    produced = {n for lw in sr.ws for n in lw.write_arrays}
    ins = [n for n in names if any(n in lw.read_arrays for lw in sr.ws) and len(sr.buf[n].shape) >= 2]
    host = {n: torch.empty(tuple(sr.buf[n].shape), dtype=sr.buf[n].dtype, pin_memory=True) for n in names}
    rm = {n: torch.empty(tuple(sr.buf[n].shape), dtype=sr.buf[n].dtype, device="cuda") for n in names}
    for n in names:
        backend.copy(rm[n], sr.buf[n])
        host[n].copy_(rm[n])
    torch.cuda.synchronize()
    # the step's results: single-kernel nests their produced array (D3Q19 dst,
    # wave4 un); multi-kernel steps every array a kernel writes
    outs = sorted(produced) if sr.multi else [sr.w.write_arrays[0]]
    sr.graphs = None                     # eager: the uploads go between wait and launch

    def roles_at(s):
        return {n: n for n in names} if sr.multi else nests.role_buffers(sr.nest, names, s)

    def upload(s, h):
        roles = roles_at(s)
        for p in ins:
            rm[p][lo:hi].copy_(host[p][lo:hi], non_blocking=True)
            backend.copy(sr.buf[roles[p]][lo:hi], rm[p][lo:hi], stream)

    def step():
        s = sr.step_no
        sr.step(stream=stream, before_launch=upload)
        roles = roles_at(s)
        for o in outs:
            backend.copy(rm[o][lo:hi], sr.buf[roles[o]][lo:hi], stream)
            host[o][lo:hi].copy_(rm[o][lo:hi], non_blocking=True)

    steps = max(3, min(args.steps, 10))
    ms = time_steps(step, steps, 2, stream, dist)
    h2d = sum(host[n][lo:hi].numel() * host[n].element_size() for n in ins)
    d2h = sum(host[o][lo:hi].numel() * host[o].element_size() for o in outs)
    total = sr.global_bytes
    return {"value": round(total / (ms * 1e-3) / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": round(ms, 3), "steps": steps,
            "path": "per rank: owned planes of the inputs, pinned host (reference layout) -> H2D -> remap -> "
                    "sharded step -> remap -> D2H of the produced planes"}


def load_traffic(kernel_name):
    """dram bytes per launch from the committed ncu summary, if present."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(kernel_name)
    except Exception:
        return None


def e2e_host_runner(args, w, k, dist):
    """Same metric through the public host-buffer API with every copy inside
    the timed region: pinned reference-layout host arrays, chunked
    H2D -> remap -> kernel -> remap -> D2H with the three overlapped on
    separate streams (paper_2306_13002_b200/pipeline_exec.HostRunner)."""
    import torch
    from paper_2306_13002_b200 import nests, pipeline_exec
    stream = torch.cuda.current_stream()
    # host inputs in the reference layout (generated on device, copied once, untimed)
    dev_rm = nests.device_inputs(w, native=False, kernel=k)
    # 0/1 int masks travel as bytes (the host buffer of D3Q19's flags is uint8)
    host = {n: torch.empty(t.shape, dtype=torch.uint8 if n == "flags" else t.dtype, pin_memory=True)
            for n, t in dev_rm.items()}
    for n, t in dev_rm.items():
        host[n].copy_(t.to(torch.uint8) if n == "flags" else t)
    del dev_rm
    torch.cuda.synchronize()
    runner = pipeline_exec.HostRunner(k, host, w.spec.range_params, chunks=args.e2e_chunks)
    sc = dict(w.scalars)
    step = lambda: runner.run(sc, args.variant, args.schedule)   # noqa: E731
    graph = None
    if not args.no_graph:
        try:
            graph = runner.capture(sc, args.variant, args.schedule)
            step = graph.replay   # same copies and launches, no host work per chunk
        except Exception as e:    # report, never hide: fall back to eager enqueue
            print(f"[bench] e2e graph capture failed, eager: {e}", file=sys.stderr)
    steps = max(3, min(args.steps, 10))
    ms = time_steps(step, steps, 2, stream, dist)
    h2d, d2h = runner.bytes_per_call()
    res = {"value": round(w.algorithmic_bytes / (ms * 1e-3) / 1e9, 3), "unit": "GB/s",
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": round(ms, 3),
           "steps": steps, "chunks": args.e2e_chunks,
           "path": "pinned host (reference layout) -> chunked H2D | acs_copy remap + acs_launch | remap + D2H, "
                   "three overlapped streams (pipeline_exec.HostRunner)"
                   + (", captured once as a CUDA graph and replayed" if graph is not None else ", eager enqueue")}
    del runner, host
    torch.cuda.empty_cache()
    return res


# ---------------------------------------------------------------------------
# per-kernel table: every nest, original vs saturated, naive vs tuned skeleton

def tune_kernel(kid, size, dtype, variant):
    """acs_tune on the BASELINE-size arrays (untimed); returns (slot, name, {slot: ms})."""
    import torch
    from paper_2306_13002_b200 import backend, nests
    w = nests.workload(kid, size, dtype=dtype)
    k = backend.Kernel.lookup(kid)
    arrs = nests.device_inputs(w, native=True, kernel=k)
    best, ms = k.tune(arrs, dict(w.scalars), variant, reps=15)
    name = k.info["schedules"][1 if dtype == "f32" else 0][best]
    del arrs
    torch.cuda.empty_cache()
    return best, name, ms


def bench_leapfrog2(kid, size, dtype, variant, slot, reps, steps=12, warmup=2):
    """wave4's two-step launch (acs_launch_leapfrog2: step 2 into a fourth buffer,
    4-buffer rotation) against the given single-step slot on the same resident
    arrays, `steps` time steps per timed sample, samples interleaved; median and
    IQR of ms per time step, GB/s of the algorithmic bytes (16 B/point/step)."""
    import torch
    from paper_2306_13002_b200 import backend, nests
    w = nests.workload(kid, size, dtype=dtype)
    k = backend.Kernel.lookup(kid)
    arrs = nests.device_inputs(w, native=True, kernel=k)
    x = backend.empty_native(k, "un", tuple(arrs["un"].shape), arrs["un"].dtype)
    sc = dict(w.scalars)
    names = list(arrs)

    def single():
        for t in range(steps):
            roles = nests.role_buffers(w.spec.nest, names, t)
            k.launch({p: arrs[r] for p, r in roles.items()}, sc, variant, slot)

    def blocked():
        b = {"u": arrs["u"], "up": arrs["up"], "un": arrs["un"], "x": x}
        for _ in range(steps // 2):
            k.launch_leapfrog2({"u": b["u"], "up": b["up"], "un": b["un"], "vel2": arrs["vel2"]}, b["x"], sc, variant)
            b = {"u": b["x"], "up": b["un"], "un": b["up"], "x": b["u"]}

    fns = [single, blocked]
    for _ in range(warmup):
        for f in fns:
            f()
    torch.cuda.synchronize()
    ev = [[] for _ in fns]
    for _ in range(reps):
        for i, f in enumerate(fns):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            f()
            b.record()
            ev[i].append((a, b))
    torch.cuda.synchronize()
    out = []
    for i in range(len(fns)):
        med, iqr = stats([a.elapsed_time(b) / steps for a, b in ev[i]])
        out.append({"ms": round(med, 4), "iqr_ms": round(iqr, 4),
                    "gbs": round(w.algorithmic_bytes / (med * 1e-3) / 1e9, 1)})
    del arrs, x
    torch.cuda.empty_cache()
    return out


def bench_configs(kid, size, dtype, sweeps, configs, reps, warmup=3):
    """Device-resident GB/s of one nest at its BASELINE size for several
    (form, schedule) configurations, each on its own resident arrays, with the
    repetitions INTERLEAVED (A B C A B C ...) so clock / power-cap drift hits
    every configuration alike; median and IQR of `reps` CUDA-event-timed steps
    each.  Buffers rotate like the nest's time loop (ping-pong / 3-level);
    a multi-sweep step (Jacobi: 100 sweeps) is one CUDA graph, replayed."""
    import torch
    from paper_2306_13002_b200 import backend, nests, stepper
    w = nests.workload(kid, size, dtype=dtype)
    k = backend.Kernel.lookup(kid)
    stream = torch.cuda.current_stream()
    steppers = []
    for variant, sched in configs:
        arrs = nests.device_inputs(w, native=True, kernel=k)
        st = stepper.Stepper(k, arrs, w.scalars, variant, sched, sweeps)
        if sweeps > 1:
            st.capture(stream)
        steppers.append(st)
    for _ in range(warmup):
        for st in steppers:
            st.step(stream)
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)] for _ in steppers]
    for r in range(reps):
        for i, st in enumerate(steppers):
            ev[i][2 * r].record(stream)
            st.step(stream)
            ev[i][2 * r + 1].record(stream)
    torch.cuda.synchronize()
    out = []
    for i in range(len(steppers)):
        ms = [ev[i][2 * r].elapsed_time(ev[i][2 * r + 1]) for r in range(reps)]
        med, iqr = stats(ms)
        gbs = w.algorithmic_bytes * sweeps / (med * 1e-3) / 1e9
        out.append({"ms": round(med, 4), "iqr_ms": round(iqr, 4), "gbs": round(gbs, 1)})
    del steppers
    torch.cuda.empty_cache()
    return out, w


# read:write array mix of every nest (smallest integers), for the mix-matched stream peak
MIX = {"jacobi7": (1, 1), "stream_collide": (1, 1), "calc1": (3, 4), "calc2": (7, 3), "calc3": (3, 2),
       "ideal_gas": (1, 1), "pdv_predict": (3, 1), "advec_cell_x": (2, 1), "wave4": (3, 1), "z_solve_lhs": (2, 3)}


def stream_peaks(mixes, elems=1 << 27, reps=10):
    """acs_stream_probe: best-of-reps GB/s of a pure R-read / W-write stream
    (1 GiB per array) for every mix — the copy peak is (1, 1); read-heavy
    nests can exceed it, write-heavy ones cannot reach it."""
    import ctypes
    from paper_2306_13002_b200 import backend
    L = backend.lib()
    L.acs_stream_probe.restype = ctypes.c_int
    L.acs_stream_probe.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                                   ctypes.POINTER(ctypes.c_float)]
    out = {}
    for r, w in sorted(set(mixes)):
        g = ctypes.c_float()
        backend._check(L.acs_stream_probe(r, w, elems, reps, ctypes.byref(g)), "acs_stream_probe")
        out[(r, w)] = round(g.value, 1)
    return out


def per_kernel_table(peak, reps):
    rows = {}
    try:
        mixpk = stream_peaks(list(MIX.values()) + [(1, 1), (1, 0)])
    except Exception as e:   # report, never hide
        mixpk = {}
        rows["stream_probe_error"] = str(e)[:200]
    if mixpk:
        # measured on this GPU in this run (acs_stream_probe; its 1R:1W is the
        # copy peak re-measured next to the driver's MEASURED_PEAKS figure)
        rows["stream_peaks"] = {"gbs": {f"{r}R:{w}W": v for (r, w), v in sorted(mixpk.items())},
                                "copy_peak_measured_peaks_json": peak}
    for kid, size, dtype, sweeps in TABLE:
        fn = kid.split(":")[1]
        row = {"size": size, "dtype": dtype, "sweeps_per_step": sweeps, "reps": reps,
               "timing": f"median and IQR of {reps} CUDA-event-timed steps per configuration, "
                         "configurations interleaved rep by rep"}
        if sweeps > 1:
            row["launch"] = f"CUDA graph of {sweeps} kernel launches per step (every form alike)"
        slots = {}
        for variant in ("accsat", "original"):
            try:
                slot, name, tms = tune_kernel(kid, size, dtype, variant)
                slots[variant] = slot
                row[f"tuned_{variant}"] = {"slot": slot, "schedule": name,
                                           "ms_per_slot": {str(s): round(v, 4) for s, v in tms.items()}}
            except Exception as e:
                row[f"tuned_{variant}"] = {"error": str(e)[:200]}
        keys = [("original", "naive", "original/naive"), ("original", slots.get("original"), "original/tuned"),
                ("original-nvcc", "naive", "original-nvcc/naive"), ("accsat", "naive", "accsat/naive"),
                ("accsat", slots.get("accsat"), "accsat/tuned")]
        if fn == "jacobi7":
            # temporal blocking (two sweeps per launch, kernels/tblock.cuh): algorithmic
            # bytes as for every form (16 B/point/sweep); DRAM bytes are about half
            keys.append(("accsat", "tb2", "accsat/tb2"))
            keys.append(("original", "tb2", "original/tb2"))
        keys = [kk for kk in keys if kk[1] is not None]
        try:
            res, w = bench_configs(kid, size, dtype, sweeps, [(v, s) for v, s, _ in keys], reps)
            for (_, _, key), r in zip(keys, res):
                r["frac"] = round(r["gbs"] / peak, 4)
                row[key] = r
        except Exception as e:  # report, never hide
            row["error"] = str(e)[:300]
            rows[fn] = row
            continue
        try:
            def ratio(a, b):
                A, B = row[a], row[b]
                band = A["iqr_ms"] / A["ms"] + B["iqr_ms"] / B["ms"]
                return {"ratio": round(B["ms"] / A["ms"], 3), "noise_band": round(band, 4),
                        "not_slower": B["ms"] / A["ms"] >= 1 - band}
            # best vs best: each form on the skeleton the tuner picked for it
            row["sat_vs_orig_best"] = ratio("accsat/tuned", "original/tuned")
            # the saturation effect alone: both forms in the same (naive) skeleton
            row["sat_vs_orig_same_skeleton"] = ratio("accsat/naive", "original/naive")
            row["sat_vs_orig_faithful"] = round(row["original/naive"]["ms"] / row["accsat/tuned"]["ms"], 3)
            row["sat_vs_nvcc_default"] = round(row["original-nvcc/naive"]["ms"] / row["accsat/tuned"]["ms"], 3)
            if "accsat/tb2" in row:
                # temporal blocking vs the best single-sweep slot: same algorithmic bytes
                # (16 B/point/sweep), about half the DRAM bytes (profiles/r02_jacobi/tb2_ncu.md)
                row["tb2_vs_tuned"] = ratio("accsat/tb2", "accsat/tuned")
                # saturation under temporal blocking: both forms through the same two-sweep kernel
                row["sat_vs_orig_tb2"] = ratio("accsat/tb2", "original/tb2")
            row["bytes_per_point"] = w.bytes_per_point
        except Exception:
            pass
        if fn == "wave4" and slots.get("accsat") is not None:
            # two leapfrog steps per launch (kernels/tbwave.cuh) vs the tuned single step,
            # interleaved on the same arrays; algorithmic bytes as for every form
            try:
                single, blocked = bench_leapfrog2(kid, size, dtype, "accsat", slots["accsat"], max(7, reps // 3))
                blocked["frac"] = round(blocked["gbs"] / peak, 4)
                row["accsat/tb2"] = blocked
                row["accsat/tuned_vs_tb2_same_run"] = single
                band = blocked["iqr_ms"] / blocked["ms"] + single["iqr_ms"] / single["ms"]
                row["tb2_vs_tuned"] = {"ratio": round(single["ms"] / blocked["ms"], 3), "noise_band": round(band, 4),
                                       "not_slower": single["ms"] / blocked["ms"] >= 1 - band}
            except Exception as e:  # report, never hide
                row["tb2_error"] = str(e)[:300]
        mix = MIX.get(fn)
        if mix and mix in mixpk and "accsat/tuned" in row and "gbs" in row["accsat/tuned"]:
            row["mix"] = f"{mix[0]}R:{mix[1]}W"
            row["mix_peak_gbs"] = round(mixpk[mix], 1)
            row["accsat/tuned"]["frac_of_mix_peak"] = round(row["accsat/tuned"]["gbs"] / mixpk[mix], 4)
        rows[fn] = row
    return rows


# ---------------------------------------------------------------------------
# CPU: the reference's own path (reported baseline, and the reference arm)

def cpu_threads(args):
    return args.cpu_threads or os.cpu_count() or 1


def mem_available():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except Exception:
        pass
    return 0


def cpu_workload(args):
    """The workloads (one per kernel of the step) the CPU runs: the full
    configured grid when the host has the memory for it (wave4 1024^3 fp32:
    17.4 GB), else a 512^3 (2-D: 4096^2) sample."""
    from paper_2306_13002_b200 import nests
    kid, dtype, _, _ = WORKLOADS[args.workload]
    ids = [kid] if isinstance(kid, str) else kid
    n = args.size
    ws = [nests.workload(k, n, dtype=dtype) for k in ids]
    dims = {}
    for w in ws:
        dims.update(w.dims)
    need = sum(int(np.prod(d)) for d in dims.values()) * (4 if dtype == "f32" else 8)
    if mem_available() < 2 * need + (8 << 30):
        n = min(args.size, 512 if len(ws[0].spec.loop_vars) == 3 else 4096)
        ws = [nests.workload(k, n, dtype=dtype) for k in ids]
    return ws, n


def cpu_inputs(ws, threads):
    """Host inputs of the step (union of its kernels' arrays, first kernel
    that declares an array fills it), generated by oracle/fill.c."""
    import cpu as oracle_cpu
    out = {}
    for w in ws:
        for n, a in oracle_cpu.host_inputs(w, threads).items():
            out.setdefault(n, a)
    return out


def run_cpu_steps(ws, variant, steps, threads, arrays):
    """Timed steps of the reference's CPU path: every kernel of the step in
    order, buffers rotating like the GPU steps (D3Q19 src <-> dst, wave4
    up <- u <- un)."""
    import cpu as oracle_cpu
    from paper_2306_13002_b200 import nests
    names = list(arrays)
    ts = []
    for s in range(steps):
        roles = nests.role_buffers(ws[0].spec.nest, names, s) if len(ws) == 1 else {n: n for n in names}
        t0 = time.perf_counter()
        for w in ws:
            a = {p.name: arrays[roles[p.name]] for p in w.spec.arrays}
            oracle_cpu.run(w.spec, a, w.scalars, variant, threads=threads, f32=w.dtype == "f32", ref=True)
        ts.append(time.perf_counter() - t0)
    return ts


def cpu_sample_desc(n, steps, ws):
    return f"{steps} steps of the {n}^{len(ws[0].spec.loop_vars)} grid" + (
        f" ({' -> '.join(w.spec.function for w in ws)} per step)" if len(ws) > 1 else "")


def cpu_baseline(args):
    import cpu as oracle_cpu
    ws, n = cpu_workload(args)
    threads = cpu_threads(args)
    arrays = cpu_inputs(ws, threads)
    nbytes = sum(w.algorithmic_bytes for w in ws)
    run_cpu_steps(ws, args.variant, 1, threads, arrays)            # first touch
    ts = run_cpu_steps(ws, args.variant, 3, threads, arrays)
    t = float(np.median(ts))
    t1 = run_cpu_steps(ws, args.variant, 1, 1, arrays)            # one core, one step
    return {"value": round(nbytes / t / 1e9, 3), "unit": "GB/s", "cores": threads,
            "value_1core": round(nbytes / t1[0] / 1e9, 3), "kind": "reference",
            "sample": f"{cpu_sample_desc(n, 3, ws)} (median) of the reference-emitted {args.variant} C "
                      "(gcc -O3 -ffp-contract=off, OpenMP over the outermost loop); value_1core: one step, one thread",
            "cpu": cpu_model()}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def reference_arm(args):
    """The reference's CPU path on this box's host cores, same metric / config
    / steps / warm-up as our arm.  Rank 0 alone runs it under torchrun."""
    rank = int(os.environ.get("RANK", "0"))
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    wl, n = cpu_workload(args)
    threads = cpu_threads(args)
    arrays = cpu_inputs(wl, threads)                             # host generator: no GPU library
    run_cpu_steps(wl, args.variant, args.warmup, threads, arrays)
    ts = run_cpu_steps(wl, args.variant, args.steps, threads, arrays)
    t = sum(ts) / len(ts)
    cfg = workload_config(args.workload, args.size, ws, args.variant)
    total = cfg["points"] * cfg["bytes_per_point"]
    # GB/s of the steps the CPU ran (a sample when the full grid does not fit)
    nbytes = sum(w.algorithmic_bytes for w in wl)
    v = nbytes / t / 1e9
    out = {"metric": METRIC, "value": round(v, 3), "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(t * 1e3 * total / nbytes, 2),
           "higher_is_better": True, "scaling": cfg["scaling"], "vs_baseline": None, "dtype": cfg["dtype"],
           "data": "synthetic (seeded SplitMix64, SURVEY.md §8d distributions; identical values to our arm)",
           "impl": "reference", "config": cfg,
           "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": threads, "kind": "reference",
                            "sample": f"{cpu_sample_desc(n, args.steps, wl)} (after {args.warmup} warm-up steps); "
                                      f"reference-emitted {args.variant} C compiled by gcc -O3 -ffp-contract=off "
                                      "(satcc wrapper mode), OpenMP over the outermost loop",
                            "cpu": cpu_model()},
           "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


if __name__ == "__main__":
    sys.exit(main() or 0)
