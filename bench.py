#!/usr/bin/env python3
"""bench.py — B200 loop-nest execution backend benchmark (one JSON line).

Workload (the N=1 line): BASELINE.json configs[1], D3Q19 lattice-Boltzmann
collide + push-stream, 256^3 fp64 (olbm-like), in the saturated form (the
reference optimizer's accsat output, frozen in tests/golden/emitted/), one
step = one stream_collide sweep src -> dst (ping-pong).  The per-kernel table
(`per_kernel`) covers every BASELINE nest in the original and saturated forms.

  value   algorithmic GB/s of the D3Q19 step with inputs resident in HBM
          (305 B per cell: 19 reads + 19 writes of 8 B + the flag byte,
          SURVEY.md §8d), whole job over all ranks.  The inputs (5.2 GB) are
          far larger than the 126 MB L2, so no L2 flush is needed between steps.
  e2e     the same metric through the public API (backend.eval_region-style
          path: pinned host buffers in the reference layout -> H2D -> AoS->SoA
          remap -> kernel -> SoA->AoS -> D2H) with the copies inside the timed
          region.

--impl reference: the reference's own CPU path for the nest — the emitted
accsat C compiled by gcc -O3 -ffp-contract=off (satcc's wrapper mode,
proj/tools/satcc_main.cpp:285-360), OpenMP over all host cores.
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
WORKLOAD_KID = "d3q19.c:stream_collide:0"

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


def dist_setup(args):
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        if args.impl == "reference":
            return rank, ws, local, None
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


def tune_kernel(kid, size, dtype, variant="accsat"):
    """acs_tune on the BASELINE-size arrays (untimed); returns (slot, name, {slot: ms})."""
    import torch
    from paper_2306_13002_b200 import backend, nests
    w = nests.workload(kid, size, dtype=dtype)
    k = backend.Kernel.lookup(kid)
    arrs = nests.device_inputs(w, native=True, kernel=k)
    best, ms = k.tune(arrs, dict(w.scalars), variant, reps=5)
    name = k.info["schedules"][1 if dtype == "f32" else 0][best]
    del arrs
    torch.cuda.empty_cache()
    return best, name, ms


def bench_kernel(kid, size, dtype, sweeps, variant, schedule, reps=5, warmup=3):
    """Device-resident GB/s of one nest at its BASELINE size (ping-pong
    where the nest has a read/write pair)."""
    import torch
    from paper_2306_13002_b200 import backend, nests
    w = nests.workload(kid, size, dtype=dtype)
    k = backend.Kernel.lookup(kid)
    arrs = nests.device_inputs(w, native=True, kernel=k)
    sc = dict(w.scalars)
    pair = {"jacobi7": ("A0", "Anext"), "d3q19": ("src", "dst")}.get(w.spec.nest)
    stream = torch.cuda.current_stream()
    state = {"t": 0}

    def step():
        for _ in range(sweeps):
            a = dict(arrs)
            t = state["t"]
            if pair and t % 2 == 1:
                a[pair[0]], a[pair[1]] = arrs[pair[1]], arrs[pair[0]]
            if w.spec.nest == "wave4":   # 3-level rotation up <- u <- un
                rot = [arrs["up"], arrs["u"], arrs["un"]]
                r = t % 3
                a["up"], a["u"], a["un"] = rot[r], rot[(r + 1) % 3], rot[(r + 2) % 3]
            k.launch(a, sc, variant, schedule, stream)
            state["t"] = t + 1

    run = step
    if sweeps > 1 and sweeps % 2 == 0 and w.spec.nest != "wave4":
        # a multi-sweep step (Jacobi: 100 ping-pong sweeps) is one CUDA graph
        # of `sweeps` kernel launches, captured once and replayed: the
        # per-launch host cost leaves the timed region, as in a real time loop
        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(stream)
        with torch.cuda.graph(g, stream=cs):
            for _ in range(sweeps):
                a = dict(arrs)
                t = state["t"]
                if pair and t % 2 == 1:
                    a[pair[0]], a[pair[1]] = arrs[pair[1]], arrs[pair[0]]
                k.launch(a, sc, variant, schedule, cs)
                state["t"] = t + 1
        stream.wait_stream(cs)
        torch.cuda.synchronize()
        run = lambda: g.replay()  # noqa: E731
    ms = time_steps(run, reps, warmup, stream)
    gbs = w.algorithmic_bytes * sweeps / (ms * 1e-3) / 1e9
    del arrs
    torch.cuda.empty_cache()
    return ms, gbs, w


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", default="accsat")
    ap.add_argument("--schedule", default="default")
    ap.add_argument("--size", type=int, default=256)
    ap.add_argument("--no-table", action="store_true", help="skip the per-kernel table")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--e2e-chunks", type=int, default=16)
    ap.add_argument("--workload", default="d3q19", choices=["d3q19", "wave4"],
                    help="d3q19: BASELINE configs[1] (N>1: weak-scaled z slabs); wave4: configs[4], "
                         "1024^3 fp32 strong-scaled over N z slabs (SURVEY.md §8e scaling metric)")
    ap.add_argument("--e2e-eager", action="store_true", help="enqueue the e2e call eagerly instead of a CUDA graph")
    ap.add_argument("--e2e-split-d2h", action="store_true", help="two download streams in the e2e pipeline")
    ap.add_argument("--e2e-ramp", action="store_true", help="smaller first/last chunks in the e2e pipeline (measured: no gain)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if isinstance(args.schedule, str) and args.schedule.isdigit():
        args.schedule = int(args.schedule)     # an explicit registered slot (0 = naive)

    if args.impl == "reference":
        return reference_arm(args)

    import torch
    from paper_2306_13002_b200 import backend, nests
    rank, ws, local, dist = dist_setup(args)
    peak, peak_kind = load_peaks()
    if args.workload == "wave4":
        return main_sharded(args, rank, ws, local, dist, peak, peak_kind)
    if ws > 1:
        return main_sharded(args, rank, ws, local, dist, peak, peak_kind)
    kid = WORKLOAD_KID
    w = nests.workload(kid, args.size)
    k = backend.Kernel.lookup(kid)
    stream = torch.cuda.current_stream()
    arrs = nests.device_inputs(w, native=True, kernel=k)
    sc = dict(w.scalars)
    tuned_slot, tuned_ms = (None, {})
    if args.schedule == "default" and args.variant != "original":
        tuned_slot, tuned_ms = k.tune(arrs, sc, args.variant, reps=5)   # untimed autotune
        arrs = nests.device_inputs(w, native=True, kernel=k)            # fresh inputs
    flip = {"f": False}
    launches = {"n": 0}

    def step():
        a = dict(arrs)
        if flip["f"]:
            a["src"], a["dst"] = arrs["dst"], arrs["src"]
        k.launch(a, sc, args.variant, args.schedule, stream)
        flip["f"] = not flip["f"]
        launches["n"] += 1

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches["n"] = 0
    with ClockSampler(local) as clk:
        ms = time_steps(step, args.steps, 0, stream, dist)
    n_launch = launches["n"]
    per_rank_bytes = w.algorithmic_bytes
    value = ws * per_rank_bytes / (ms * 1e-3) / 1e9
    achieved = per_rank_bytes / (ms * 1e-3) / 1e9

    out = {"metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": ws,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded SplitMix64, SURVEY.md §8d distributions; generated in HBM)",
           "config": {"workload": "D3Q19 lattice-Boltzmann collide+stream (olbm-like) fp64, one sweep per step",
                      "grid": [args.size] * 3, "form": args.variant, "schedule": args.schedule,
                      "layout": "q-major SoA in HBM", "l2": "inputs 5.2 GB >> 126 MB L2 (no flush needed)",
                      "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
                      "bytes_per_point": w.bytes_per_point, "points": w.points},
           "gpu_launches": n_launch}
    out["roofline"] = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                       "frac": round(achieved / peak, 4), "peak_kind": peak_kind,
                       "traffic": load_traffic("stream_collide"),
                       "kernel": f"stream_collide {args.variant}: " + (
                           k.info["schedules"][0][tuned_slot] if tuned_slot is not None
                           else (k.info["schedules"][0][args.schedule] if isinstance(args.schedule, int)
                                 else args.schedule))}
    out["config"]["tuned"] = {"slot": tuned_slot, "ms_per_slot": {str(s): round(v, 4) for s, v in tuned_ms.items()}}
    out["clocks"] = clk.summary()

    del arrs
    torch.cuda.empty_cache()
    if not args.no_e2e:
        out["e2e"] = e2e_d3q19(args, w, k, dist)
    if not args.no_table and ws == 1:
        out["per_kernel"] = per_kernel_table(peak)
    if rank == 0 and ws == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(w, args)
    if dist:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out))


def main_sharded(args, rank, ws, local, dist, peak, peak_kind):
    """N GPUs.  d3q19: the domain is slab-sharded along z, 256 planes per rank
    (weak scaling: global grid 256 x 256 x 256N); the pushes that cross a slab
    face are written straight into the neighbour's distribution array.
    wave4 (--workload wave4, any N): the 1024^3 fp32 grid split into N z
    slabs (strong scaling); the new boundary planes of `un` are written into
    the neighbours' halos.  Both over NVLink (CUDA IPC peer memory, from
    inside the kernel), steps ordered by device-side flags."""
    import torch
    from paper_2306_13002_b200 import backend, nests, shard
    wave = args.workload == "wave4"
    kid = "wave4.c:wave4:0" if wave else WORKLOAD_KID
    gsize = 1024 if args.size == 256 and wave else args.size
    size = (gsize, gsize, gsize) if wave else (args.size * ws, args.size, args.size)
    sr = shard.SlabRank(kid, size, ws, rank, dtype="f32" if wave else "f64", variant=args.variant,
                        schedule=args.schedule)
    stream = torch.cuda.current_stream()
    tuned = None
    if args.schedule == "default" and args.variant != "original":
        tuned, _ = sr.k.tune(sr.buf, dict(sr.w.scalars), args.variant, reps=5)   # untimed
        sr.schedule = tuned
        sr.refill()
    torch.cuda.synchronize()
    peer_error = None
    if ws > 1:
        exp = [None] * ws
        dist.all_gather_object(exp, sr.export())
        try:
            sr.connect_ipc(exp[rank - 1] if rank > 0 else None, exp[rank + 1] if rank < ws - 1 else None)
        except Exception as e:     # no peer access between these GPUs
            peer_error = str(e)[:200]
        errs = [None] * ws
        dist.all_gather_object(errs, peer_error)
        if any(errs):
            # every rank falls back together: slabs without neighbours (no
            # halo exchange) — reported as such, never as the sharded number
            sr.close()
            sr.lo_ptr, sr.hi_ptr, sr.lo_flag, sr.hi_flag = {}, {}, None, None
            peer_error = next(e for e in errs if e)
            print(f"[bench] rank {rank}: peer memory unavailable ({peer_error}); running slabs as replicas",
                  file=sys.stderr)
        dist.barrier()
    launches = {"n": 0}

    def step():
        sr.step(stream=stream)
        launches["n"] += 1 + (1 if sr.step_no > 1 and (sr.lo_ptr or sr.hi_ptr) else 0) + (1 if sr.lo_flag or sr.hi_flag else 0)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches["n"] = 0
    with ClockSampler(local) as clk:
        ms = time_steps(step, args.steps, 0, stream, dist)
    local_bytes = sr.w.algorithmic_bytes
    total_bytes = sr.gw.algorithmic_bytes if wave else ws * local_bytes
    value = total_bytes / (ms * 1e-3) / 1e9
    if wave:
        cfg = {"workload": "seismic wave4 4th-order 3-D wave propagation fp32, one step per step (3-level rotation)",
               "grid": [gsize] * 3, "per_rank_planes": sr.plan.owned(rank)[1] - sr.plan.owned(rank)[0],
               "form": args.variant, "schedule": args.schedule, "tuned_slot": tuned,
               "parallelism": f"z-slab sharding x{ws} (strong scaling), fused peer-memory halo write-through + "
                              "device flags",
               "layout": "row-major, padded pitch", "l2": "inputs >> L2 (no flush needed)",
               "bytes_per_point": sr.w.bytes_per_point}
    else:
        cfg = {"workload": "D3Q19 lattice-Boltzmann collide+stream (olbm-like) fp64, one sweep per step",
               "grid": [args.size, args.size, args.size * ws], "per_rank_grid": [args.size] * 3,
               "form": args.variant, "schedule": args.schedule, "tuned_slot": tuned,
               "parallelism": f"z-slab sharding x{ws}, fused peer-memory push exchange + device flags",
               "layout": "q-major SoA in HBM", "l2": "inputs >> L2 (no flush needed)",
               "bytes_per_point": sr.w.bytes_per_point}
    out = {"metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
           "scaling": "strong" if wave else "weak", "vs_baseline": None, "dtype": "f32" if wave else "f64",
           "data": "synthetic (seeded SplitMix64, SURVEY.md §8d distributions; generated in HBM)",
           "config": cfg, "gpu_launches": launches["n"]}
    if peer_error:
        out["config"]["parallelism"] = f"replicas x{ws}: peer memory unavailable, no halo exchange ({peer_error})"
    achieved = local_bytes / (ms * 1e-3) / 1e9
    out["roofline"] = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                       "frac": round(achieved / peak, 4), "peak_kind": peak_kind,
                       "traffic": load_traffic("wave4_f32" if wave else "stream_collide"),
                       "kernel": ("wave4_f32 " if wave else "stream_collide ") + args.variant + " (sharded, per rank)"}
    out["clocks"] = clk.summary()
    if not args.no_e2e:
        if ws == 1:
            # one slab: the overlapped host-buffer pipeline (as for the D3Q19 line)
            sr.close()
            del sr.buf
            torch.cuda.empty_cache()
            out["e2e"] = e2e_d3q19(args, sr.gw, sr.k, dist)
        else:
            out["e2e"] = e2e_sharded(args, sr, dist, ws)
    sr.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out))
    return 0


def e2e_sharded(args, sr, dist, ws):
    """Per rank per step: its slab's reference-layout host buffers -> device ->
    remap -> sharded step (with the peer exchange) -> remap -> host."""
    import torch
    from paper_2306_13002_b200 import backend, shard
    stream = torch.cuda.current_stream()
    names = [a.name for a in sr.w.spec.arrays]
    host = {n: torch.empty(tuple(sr.buf[n].shape), dtype=sr.buf[n].dtype, pin_memory=True) for n in names}
    rm = {n: torch.empty(tuple(sr.buf[n].shape), dtype=sr.buf[n].dtype, device="cuda") for n in names}
    for n in names:
        backend.copy(rm[n], sr.buf[n])
        host[n].copy_(rm[n])
    torch.cuda.synchronize()

    out_name = sr.w.write_arrays[0]      # the produced array: D3Q19 dst, wave4 un

    def step():
        roles = shard.role_buffers(sr.nest, names, sr.step_no)
        for p in names:
            rm[p].copy_(host[p], non_blocking=True)
            backend.copy(sr.buf[roles[p]], rm[p], stream)
        sr.step(stream=stream)
        backend.copy(rm[out_name], sr.buf[roles[out_name]], stream)
        host[out_name].copy_(rm[out_name], non_blocking=True)

    steps = max(3, min(args.steps, 10))
    ms = time_steps(step, steps, 2, stream, dist)
    h2d = sum(host[n].numel() * host[n].element_size() for n in names)
    d2h = host[out_name].numel() * host[out_name].element_size()
    total = sr.gw.algorithmic_bytes if args.workload == "wave4" else ws * sr.w.algorithmic_bytes
    return {"value": round(total / (ms * 1e-3) / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": round(ms, 3), "steps": steps,
            "path": "per rank: pinned host slab (reference AoS) -> H2D -> remap -> sharded acs_launch -> remap -> D2H"}


def load_traffic(kernel_name):
    """dram bytes per launch from the committed ncu summary, if present."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(kernel_name)
    except Exception:
        return None


def e2e_d3q19(args, w, k, dist):
    """Same metric through the public host-buffer API with every copy inside
    the timed region: pinned reference-layout (AoS) host arrays, chunked
    H2D -> remap -> kernel -> remap -> D2H with the three overlapped on
    separate streams (paper_2306_13002_b200/pipeline_exec.HostRunner)."""
    import torch
    from paper_2306_13002_b200 import nests, pipeline_exec
    stream = torch.cuda.current_stream()
    # host inputs in the reference layout (generated on device, copied once, untimed)
    dev_rm = nests.device_inputs(w, native=False, kernel=k)
    host = {n: torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for n, t in dev_rm.items()}
    for n, t in dev_rm.items():
        host[n].copy_(t)
    del dev_rm
    torch.cuda.synchronize()
    runner = pipeline_exec.HostRunner(k, host, w.spec.range_params, chunks=args.e2e_chunks, ramp=args.e2e_ramp)
    runner.split_d2h = args.e2e_split_d2h
    sc = dict(w.scalars)

    def step():
        runner.run(sc, args.variant, args.schedule)

    graph = None
    if not args.e2e_eager:
        try:
            graph = runner.capture(sc, args.variant, args.schedule)
            step = graph.replay   # noqa: F811 — same copies and launches, no host work per chunk
        except Exception as e:    # report, never hide: fall back to eager enqueue
            print(f"[bench] e2e graph capture failed, eager: {e}", file=sys.stderr)
    steps = max(3, min(args.steps, 10))
    ms = time_steps(step, steps, 2, stream, dist)
    ws = dist.get_world_size() if dist else 1
    h2d, d2h = runner.bytes_per_call()
    res = {"value": round(ws * w.algorithmic_bytes / (ms * 1e-3) / 1e9, 3), "unit": "GB/s",
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": round(ms, 3),
           "steps": steps, "chunks": args.e2e_chunks,
           "path": "pinned host (reference AoS layout) -> chunked H2D | acs_copy remap + acs_launch | remap + D2H, "
                   "three overlapped streams (pipeline_exec.HostRunner)"
                   + (", captured once as a CUDA graph and replayed" if graph is not None else ", eager enqueue")}
    del runner, host
    torch.cuda.empty_cache()
    return res


def per_kernel_table(peak):
    rows = {}
    for kid, size, dtype, sweeps in TABLE:
        fn = kid.split(":")[1]
        row = {"size": size, "dtype": dtype, "sweeps_per_step": sweeps}
        if sweeps > 1:
            row["launch"] = f"CUDA graph of {sweeps} kernel launches per step (every form alike)"
        try:
            slot, name, tms = tune_kernel(kid, size, dtype, "accsat")
            row["tuned"] = {"slot": slot, "schedule": name, "ms_per_slot": {str(s): round(v, 4) for s, v in tms.items()}}
        except Exception as e:
            row["tuned"] = {"error": str(e)[:200]}
        for variant, sched in (("original", "naive"), ("original-nvcc", "naive"), ("accsat", "naive"),
                               ("accsat", "default")):
            try:
                ms, gbs, w = bench_kernel(kid, size, dtype, sweeps, variant, sched, reps=5)
                row[f"{variant}/{sched}"] = {"ms": round(ms, 4), "gbs": round(gbs, 1), "frac": round(gbs / peak, 4)}
            except Exception as e:  # report, never hide
                row[f"{variant}/{sched}"] = {"error": str(e)[:200]}
        try:
            row["sat_vs_orig_speedup"] = round(row["accsat/default"]["gbs"] / row["original/naive"]["gbs"], 3)
            row["sat_vs_nvcc_default_speedup"] = round(row["accsat/default"]["gbs"] / row["original-nvcc/naive"]["gbs"], 3)
            # the saturation effect alone: both forms in the same (naive) skeleton
            row["sat_vs_orig_same_skeleton"] = round(row["accsat/naive"]["gbs"] / row["original/naive"]["gbs"], 3)
            row["bytes_per_point"] = w.bytes_per_point
        except Exception:
            pass
        rows[fn] = row
    return rows


def cpu_threads(args):
    return args.cpu_threads or os.cpu_count() or 1


def run_cpu_steps(w, variant, steps, threads, arrays=None):
    """Timed steps of the reference's CPU path, buffers rotating like the GPU
    steps (D3Q19 src <-> dst, wave4 up <- u <- un)."""
    import cpu as oracle_cpu
    from paper_2306_13002_b200 import shard
    if arrays is None:
        arrays = host_inputs_via_gpu(w)
    names = list(arrays)
    ts = []
    for s in range(steps):
        roles = shard.role_buffers(w.spec.nest, names, s)
        a = {p: arrays[roles[p]] for p in names}
        t0 = time.perf_counter()
        oracle_cpu.run(w.spec, a, w.scalars, variant, threads=threads, f32=w.dtype == "f32")
        ts.append(time.perf_counter() - t0)
    return ts, arrays


def host_inputs_via_gpu(w):
    """Reference-layout host inputs: generated on the device when a GPU is
    present (fast), else with numpy (identical values)."""
    from paper_2306_13002_b200 import nests
    try:
        import torch
        if torch.cuda.is_available():
            dev = nests.device_inputs(w, native=False)
            out = {n: t.cpu().numpy() for n, t in dev.items()}
            del dev
            torch.cuda.empty_cache()
            return out
    except Exception:
        pass
    return nests.make_inputs(w)


def cpu_baseline(w, args):
    threads = cpu_threads(args)
    ts, arrays = run_cpu_steps(w, "accsat", 3, threads)
    t = float(np.median(ts))
    t1, _ = run_cpu_steps(w, "accsat", 1, 1, arrays)      # one core, one sweep
    return {"value": round(w.algorithmic_bytes / t / 1e9, 3), "unit": "GB/s", "cores": threads,
            "value_1core": round(w.algorithmic_bytes / t1[0] / 1e9, 3),
            "kind": "reference",
            "sample": f"3 full {w.dims['flags']} D3Q19 sweeps of the reference-emitted accsat C "
                      f"(gcc -O3 -ffp-contract=off, OpenMP over z), median",
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
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2306_13002_b200 import nests
    wave = args.workload == "wave4"
    # wave4: a bounded 512^3 sample of the 1024^3 workload (4 x 0.54 GB host arrays)
    w = nests.workload("wave4.c:wave4:0", 512 if args.size == 256 else min(args.size, 512), dtype="f32") if wave \
        else nests.workload(WORKLOAD_KID, args.size)
    threads = cpu_threads(args)
    arrays = host_inputs_via_gpu(w)
    run_cpu_steps(w, args.variant, 1, threads, arrays)       # warm-up (first touch)
    steps = max(1, min(args.steps, 10))
    ts, _ = run_cpu_steps(w, args.variant, steps, threads, arrays)
    t = sum(ts) / len(ts)
    v = w.algorithmic_bytes / t / 1e9
    out = {"metric": METRIC, "value": round(v, 3), "unit": "GB/s", "n_gpus": args.gpus, "steps": steps,
           "warmup": 1, "ms_per_step": round(t * 1e3, 2), "higher_is_better": True,
           "scaling": "strong" if wave else "weak",
           "vs_baseline": None, "dtype": "f32" if wave else "f64", "data": "synthetic (seeded SplitMix64, identical inputs)",
           "impl": "reference",
           "config": ({"workload": "seismic wave4 4th-order 3-D wave propagation fp32, one step per step "
                                   "(3-level rotation)", "grid": [1024] * 3,
                       "form": args.variant} if wave else
                      {"workload": "D3Q19 lattice-Boltzmann collide+stream (olbm-like) fp64, one sweep per step",
                       "grid": [args.size] * 3, "form": args.variant}),
           "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": threads, "kind": "reference",
                            "sample": (f"{steps} steps on a {round(w.points ** (1 / 3))}^3 sample" if wave
                                       else f"{steps} full sweeps") +
                                      f"; reference-emitted {args.variant} C compiled by gcc "
                                      "-O3 -ffp-contract=off (satcc wrapper mode), OpenMP over z",
                            "cpu": cpu_model()},
           "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


if __name__ == "__main__":
    sys.exit(main() or 0)
