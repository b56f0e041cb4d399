#!/usr/bin/env python3
"""Benchmark of the tropical hot path on B200 (driver contract: one JSON line).

Default workload (BASELINE.json configs[1]): min-plus GEMM, n = 16384, int32
storage ("DPX"), operands uniform integers in [-1000, 1000] with 25 % Infinity
(the C2 recipe of SURVEY §8(d)).  One step = one C = A ⊗ B through the
product path (btas_gemm: screen, packing, GEMM kernel) with A, B resident in
HBM.  Metric: G(add,min)/s = n^3 / step time / 1e9.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                    [--workload gemm|gemm_f32|gemm_f32_real|fw|apsp|matvec|ewadd|graph] [--n N]

N > 1 (launched by torchrun, one rank per GPU): every rank runs its own
independent GEMM of the same size — the GEMM shards into independent output
blocks, there is no data-path collective (weak scaling); the elapsed time is
the max over ranks.

Keys beyond the base contract:
  roofline      the GEMM kernel's achieved pair rate (CUDA events around the
                kernel launches, on the launching stream) vs the live ceiling
                of its instruction mix (btas_probe_ceiling: pairs/clk/SM x SMs
                x the SM clock sampled during the timed region)
  cpu_baseline  the reference algorithm restated in NumPy (oracle/tropical.py,
                "port": the reference's broadcast-add + reduce tiles on a
                thread pool), timed on this host on a sampled row block
  e2e           the same metric through the public API from pinned host
                buffers: TropicalMatrix(host) x2 + matmul + D2H of the result
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "tropical GEMM G(add,min)/s at n=16384"
UNIT = "Gpair/s"


def parse():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[1])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="gemm",
                    choices=["gemm", "gemm_f32", "gemm_f32_real", "fw", "apsp", "matvec", "ewadd", "graph"])
    ap.add_argument("--batch", type=int, default=1, help="vectors per matvec (config C5: 1, 2, 4, 8)")
    ap.add_argument("--n", type=int, default=0, help="problem size (default per workload)")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-apsp", action="store_true", help="skip the APSP C4 measurement of the default run")
    ap.add_argument("--apsp-n", type=int, default=65536, help="APSP C4 size inside the default run")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------
class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# synthetic inputs
# ---------------------------------------------------------------------------
def gemm_inputs(n, dtype, device, seed, real=False):
    """C2 recipe: integers in [-1000, 1000] (or reals rounded to f32), 25 % Infinity."""
    import torch

    import paper_1701_04733_b200 as bt

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    if real:
        sym = (torch.rand((n, n), generator=g, device=device, dtype=torch.float32) * 2000.0 - 1000.0)
    else:
        sym = torch.randint(-1000, 1001, (n, n), generator=g, device=device, dtype=torch.int32).to(torch.float32)
    inf_mask = torch.rand((n, n), generator=g, device=device) < 0.25
    sym[inf_mask] = math.inf
    m = bt.TropicalMatrix(bt.SemiringKind.MIN_PLUS, sym, dtype=dtype, device=device)
    return m, sym


# ---------------------------------------------------------------------------
# CPU baseline: the reference algorithm (NumPy port), sampled rows
# ---------------------------------------------------------------------------
def cpu_baseline_gemm(x_sym_rows, y_sym, storage, integer, budget_rows):
    from oracle import tropical as ot

    cores = len(os.sched_getaffinity(0))
    xo = ot.orient(ot.MIN, x_sym_rows[:budget_rows])
    yo = ot.orient(ot.MIN, y_sym)
    ot.matmul(xo[:1], yo[:, :256], ot.MIN, storage, integer)  # warm-up
    t = time.perf_counter()
    ot.matmul(xo, yo, ot.MIN, storage, integer, tile_rows=4, tile_cols=128, workers=cores)
    dt = time.perf_counter() - t
    pairs = xo.shape[0] * yo.shape[0] * yo.shape[1]
    return pairs / dt / 1e9, cores, dt, pairs


def cpu_sample_rows():
    cores = len(os.sched_getaffinity(0))
    return int(min(256, max(8, 4 * cores)))


# ---------------------------------------------------------------------------
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, rank, world)

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    if args.workload in ("fw", "apsp"):
        return apsp_arm(args, rank, world, dev)
    if args.workload in ("matvec", "ewadd"):
        return hbm_arm(args, rank, world, dev)
    if args.workload == "graph":
        return graph_arm(args, rank, world, dev)

    import paper_1701_04733_b200 as bt
    from paper_1701_04733_b200 import _lib

    n = args.n or 16384
    dtype, real, wl = {
        "gemm": (torch.int32, False, f"minplus_gemm_n{n}_i32"),
        "gemm_f32": (torch.float32, False, f"minplus_gemm_n{n}_f32_integer"),
        "gemm_f32_real": (torch.float32, True, f"minplus_gemm_n{n}_f32_real"),
    }[args.workload]

    # ------------------------------------------------------------- timed run
    from paper_1701_04733_b200 import matrix as bm

    seed = 0xB2000001 + 7919 * rank
    x, xs = gemm_inputs(n, dtype, dev, seed, real)
    y, ys = gemm_inputs(n, dtype, dev, seed + 1, real)
    integer = x.integer and y.integer
    out = torch.empty((n, n), dtype=dtype, device=dev)
    flags = None
    for _ in range(max(3, args.warmup)):
        _, flags = bm._gemm(x.data, y.data, bt.SemiringKind.MIN_PLUS, integer, out=out)
    torch.cuda.synchronize()
    path_bits = int(flags[_lib.FLAG_PATH].item())
    path = [name for p, name in _lib.PATH_NAMES.items() if path_bits & (1 << p)][0]

    stream = torch.cuda.current_stream(dev)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    _lib.gemm_timing(True)
    with ClockSampler(local) as clocks:
        start.record(stream)
        for _ in range(args.steps):
            bm._gemm(x.data, y.data, bt.SemiringKind.MIN_PLUS, integer, out=out)
        stop.record(stream)
        torch.cuda.synchronize()
    kernel_ms, kernel_count = _lib.gemm_timing_read()
    _lib.gemm_timing(False)
    elapsed_ms = start.elapsed_time(stop)
    if world > 1:
        t = torch.tensor([elapsed_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
        dist.barrier()
    pairs = float(n) ** 3
    value = pairs * args.steps * world / (elapsed_ms * 1e-3) / 1e9
    clk = clocks.summary()

    # roofline: the GEMM kernel vs the live ceiling of its instruction mix
    mix = {"s16x2": 2, "fast32": 1 if dtype == torch.int32 else 0}.get(path, 0)
    probe = _lib.probe_ceiling(mix)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    sm_mhz = clk["sm_mhz"] or probe["sm_mhz"]
    peak = probe["pairs_per_clk_sm"] * nsm * sm_mhz * 1e6 / 1e12
    achieved = pairs / (kernel_ms / kernel_count * 1e-3) / 1e12
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get(wl)
    roofline = {
        "bound": "alu",
        "achieved": round(achieved, 3),
        "peak": round(peak, 3),
        "unit": "Tpair/s",
        "frac": round(achieved / peak, 4),
        "traffic": traffic,
        "kernel": {"s16x2": "tropical_gemm_kernel<MixS16>", "fast32": "tropical_gemm_kernel<MixI32|MixF32>"}.get(
            path, path),
        "kernel_ms": round(kernel_ms / kernel_count, 3),
        "step_ms": round(elapsed_ms / args.steps, 3),
        "peak_mix_pairs_per_clk_sm": round(probe["pairs_per_clk_sm"], 2),
        "peak_sm_mhz": sm_mhz,
        "peak_source": "btas_probe_ceiling (live register/LDS microbenchmark of the same add-min instruction mix) "
                       "x SMs x median SM clock during the timed region",
        "peak_at_max_clock": round(probe["pairs_per_clk_sm"] * nsm * 1965e6 / 1e12, 3),
    }

    result = {
        "metric": METRIC,
        "value": round(value, 1),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(3, args.warmup),
        "ms_per_step": round(elapsed_ms / args.steps, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": {torch.int32: "i32", torch.float32: "f32"}[dtype],
        "data": "synthetic",
        "config": {
            "workload": wl,
            "n": n,
            "operands": "uniform reals in [-1000,1000) rounded to f32" if real else "uniform integers in [-1000,1000]",
            "infinity_fraction": 0.25,
            "kernel_path": path,
            "l2": "operands 1 GiB each >> 126 MB L2; no flush needed",
            "parallelism": f"dp{world} (independent GEMM per GPU)",
        },
        "roofline": roofline,
        "gpu_launches": args.steps * (11 if integer else 8),
        "clocks": clk,
    }

    if traffic is not None:
        roofline["traffic_note"] = ("dram bytes per launch (ncu --set full); above the compulsory 2-3 GB because "
                                    "L2 serves ~90 % of the 128 GB of tile loads — HBM runs at ~2 % of peak")

    # ------------------------------------------------------------- e2e (public API, host buffers)
    if not args.no_e2e:
        try:
            e2e = e2e_gemm(n, dtype, xs, ys, dev, steps=max(3, args.steps))
        except (RuntimeError, MemoryError) as exc:  # e.g. pinned host memory exhausted: keep the line
            e2e = {"error": f"{type(exc).__name__}: {exc}"[:300], "ms_per_step": float("nan")}
        if world > 1:  # whole job: every rank's steps over the slowest rank's time
            t = torch.tensor([e2e["ms_per_step"]], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e["ms_per_step"] = round(float(t.item()), 2)
            e2e["value"] = round(float(n) ** 3 * world / (e2e["ms_per_step"] * 1e-3) / 1e9, 1)
        result["e2e"] = e2e

    # ------------------------------------------------------------- other kernel paths (N = 1 only)
    if not args.no_variants and args.workload == "gemm" and world == 1:
        result["variants"] = variants(n, dev, rank)

    # ------------------------------------------------------------- CPU baseline (rank 0, N = 1)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rows = cpu_sample_rows()
        storage = {torch.int32: "i32", torch.float32: "f32"}[dtype]
        xh = xs[:rows].double().cpu().numpy()
        yh = ys.double().cpu().numpy()
        v, cores, secs, spairs = cpu_baseline_gemm(xh, yh, storage, integer, rows)
        result["cpu_baseline"] = {
            "value": round(v, 4), "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{rows} rows x {n} x {n} ({spairs:.3g} pairs, {secs:.1f} s) of the same operands; "
                      "NumPy restatement of btas.matmul (_product_tile broadcast-add + reduce, thread pool of "
                      f"{cores} workers)",
        }
    # ------------------------------------------------------------- APSP C4 (north-star scaling row)
    if not args.no_apsp and args.workload == "gemm":
        del x, y, out, xs, ys
        torch.cuda.empty_cache()

        def give_up():  # a stuck exchange must not cost the GEMM line
            result["apsp_c4"] = {"error": f"timed out after {APSP_WATCHDOG_S} s"}
            if rank == 0:
                print(json.dumps(result), flush=True)
            os._exit(0)

        timer = threading.Timer(APSP_WATCHDOG_S, give_up)
        timer.daemon = True
        timer.start()
        try:
            result["apsp_c4"] = apsp_c4(args.apsp_n, rank, world, dev)
        except Exception as exc:  # report, keep the GEMM line
            result["apsp_c4"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        finally:
            timer.cancel()
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


APSP_WATCHDOG_S = 420


def apsp_c4(n, rank, world, dev):
    """BASELINE config C4 inside the default run: repeated-squaring APSP of
    the n = 65536 instance graph_to_matrix(random_graph(n, 0.5, (1, 100),
    instance_seed(1, n))) in fp32, on 1 GPU or row-sharded over the ranks
    (all-gather fused into the GEMM epilogue over symmetric memory, NCCL
    fallback).  One timed solve after a small warm-up solve; device time,
    max over ranks.  "scaling": strong (the instance is fixed)."""
    import torch
    import torch.distributed as dist

    import paper_1701_04733_b200 as bt
    from paper_1701_04733_b200.graphs import instance_seed, random_graph_matrix

    if world > 1:
        from paper_1701_04733_b200.sharded import apsp_by_squaring_distributed as solver
    else:
        solver = bt.apsp_by_squaring
    solver(random_graph_matrix(2048, 0.5, (1, 100), instance_seed(1, 2048), dtype=torch.float32, device=dev))
    adj = random_graph_matrix(n, 0.5, (1, 100), instance_seed(1, n), dtype=torch.float32, device=dev)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    rep = solver(adj)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    d = rep.distances.dist.data
    checksum = 0  # of the finite distances (inf -> -1), identical for every N
    for r0 in range(0, n, 4096):
        blk = d[r0:r0 + 4096]
        blk = torch.where(torch.isfinite(blk), blk, torch.full_like(blk, -1)).to(torch.int64)
        checksum = (checksum + int(blk.sum().item())) % (1 << 61)
    out = {"metric": f"APSP time n={n}", "value": round(ms / 1e3, 3), "unit": "s", "higher_is_better": False,
           "n_gpus": world, "scaling": "strong", "dtype": "f32",
           "config": {"workload": f"apsp_squaring_n{n}_f32", "graph": "random_graph p=0.5 weights 1..100",
                      "instance_seed": "instance_seed(1, n)"},
           "multiplications": rep.multiplications_performed, "negative_cycle": rep.negative_cycle,
           "distance_checksum": checksum,
           "tpairs_per_s": round(float(n) ** 3 * rep.multiplications_performed / (ms * 1e-3) / 1e12, 2)}
    if world > 1:
        out["exchange"] = os.environ.get("BTAS_EXCHANGE", "auto")
    del adj, rep, d
    torch.cuda.empty_cache()
    return out


def e2e_gemm(n, dtype, xs, ys, dev, steps):
    """Public API end to end, every step: host symbolic operands (pinned f32)
    -> two TropicalMatrix constructions (H2D + validation/ingest on the GPU)
    -> matmul -> D2H of the result storage into pinned memory.

    Reported twice: `serial_ms_per_step` runs one step at a time; the headline
    runs the same calls on three CUDA streams (copy-in / compute / copy-out,
    double-buffered host outputs) so step i's uploads and step i-1's download
    overlap step i-1's / i's GEMM — a throughput pipeline over independent
    steps, each still paying its full H2D and D2H."""
    import torch

    import paper_1701_04733_b200 as bt

    hx = xs.cpu().pin_memory()
    hy = ys.cpu().pin_memory()
    hout = [torch.empty((n, n), dtype=dtype).pin_memory() for _ in range(2)]
    MIN = bt.SemiringKind.MIN_PLUS

    def serial_step():
        X = bt.TropicalMatrix(MIN, hx, dtype=dtype, device=dev)
        Y = bt.TropicalMatrix(MIN, hy, dtype=dtype, device=dev)
        Z = bt.matmul(X, Y)
        hout[0].copy_(Z.data, non_blocking=True)
        torch.cuda.synchronize()

    serial_step()
    t = time.perf_counter()
    for _ in range(steps):
        serial_step()
    serial = (time.perf_counter() - t) / steps

    s_in, s_comp, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def pipelined(k):
        for i in range(k):
            with torch.cuda.stream(s_in):
                # both uploads first: the validating ingest kernels queue
                # behind the running GEMM, so the host must not block on X's
                # validation before Y's upload has been issued
                dx = hx.to(dev, non_blocking=True)
                dy = hy.to(dev, non_blocking=True)
                X = bt.TropicalMatrix(MIN, dx, dtype=dtype, device=dev)
                Y = bt.TropicalMatrix(MIN, dy, dtype=dtype, device=dev)
            s_comp.wait_stream(s_in)
            with torch.cuda.stream(s_comp):
                X.data.record_stream(s_comp)
                Y.data.record_stream(s_comp)
                Z = bt.matmul(X, Y)
            s_out.wait_stream(s_comp)
            with torch.cuda.stream(s_out):
                Z.data.record_stream(s_out)
                hout[i % 2].copy_(Z.data, non_blocking=True)
        torch.cuda.synchronize()

    pipelined(2)
    t = time.perf_counter()
    pipelined(steps)
    dt = (time.perf_counter() - t) / steps
    return {
        "value": round(float(n) ** 3 / dt / 1e9, 1),
        "unit": UNIT,
        "h2d_bytes_per_step": 2 * n * n * 4,
        "d2h_bytes_per_step": n * n * torch.tensor([], dtype=dtype).element_size(),
        "ms_per_step": round(dt * 1e3, 2),
        "serial_ms_per_step": round(serial * 1e3, 2),
        "serial_value": round(float(n) ** 3 / serial / 1e9, 1),
        "steps": steps,
        "path": "pinned f32 host operands -> H2D -> TropicalMatrix(validate+ingest) x2 -> matmul -> result D2H "
                "(pinned); 3-stream pipeline over steps",
    }


def variants(n, dev, rank):
    """The other kernel paths on the same size (fewer steps)."""
    import torch

    import paper_1701_04733_b200 as bt
    from paper_1701_04733_b200 import _lib
    from paper_1701_04733_b200 import matrix as bm

    out = {}
    cases = {
        "f32_integer_valued": (torch.float32, False, 1000),
        "f32_real_valued": (torch.float32, True, 1000),
        "i32_wide_range": (torch.int32, False, 10**6),
        "f64_integer_wide_range": (torch.float64, False, 10**6),  # the reference's default dtype
    }
    for name, (dtype, real, rng) in cases.items():
        g = torch.Generator(device=dev)
        g.manual_seed(0xB2000002 + rank)
        mats = []
        for _ in range(2):
            if real:
                sym = torch.rand((n, n), generator=g, device=dev) * 2000.0 - 1000.0
            else:
                sym = torch.randint(-rng, rng + 1, (n, n), generator=g, device=dev, dtype=torch.int32).to(torch.float32)
            sym[torch.rand((n, n), generator=g, device=dev) < 0.25] = math.inf
            mats.append(bt.TropicalMatrix(bt.SemiringKind.MIN_PLUS, sym, dtype=dtype, device=dev))
            del sym
        x, y = mats
        integer = x.integer and y.integer
        o = torch.empty((n, n), dtype=dtype, device=dev)
        _, flags = bm._gemm(x.data, y.data, bt.SemiringKind.MIN_PLUS, integer, out=o)
        torch.cuda.synchronize()
        bits = int(flags[_lib.FLAG_PATH].item())
        path = [nm for p, nm in _lib.PATH_NAMES.items() if bits & (1 << p)][0]
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        _lib.gemm_timing(True)
        s.record()
        for _ in range(3):
            bm._gemm(x.data, y.data, bt.SemiringKind.MIN_PLUS, integer, out=o)
        e.record()
        torch.cuda.synchronize()
        kms, kc = _lib.gemm_timing_read()
        _lib.gemm_timing(False)
        ms = s.elapsed_time(e) / 3
        mix = {"s16x2": 2, "i32f64": 1}.get(path, 1 if dtype == torch.int32 else 0)
        probe = _lib.probe_ceiling(mix)
        nsm = torch.cuda.get_device_properties(dev).multi_processor_count
        peak = probe["pairs_per_clk_sm"] * nsm * probe["sm_mhz"] * 1e6 / 1e12
        ach = float(n) ** 3 / (kms / kc * 1e-3) / 1e12
        out[name] = {"value": round(float(n) ** 3 / (ms * 1e-3) / 1e9, 1), "unit": UNIT, "kernel_path": path,
                     "kernel_tpairs": round(ach, 3), "peak_tpairs_probe_clock": round(peak, 3),
                     "frac": round(ach / peak, 4)}
        del x, y, o, mats
        torch.cuda.empty_cache()
    return out


def apsp_arm(args, rank, world, dev):
    """FW (C3) / squaring (C1, C4) timing on one GPU (replicas for N > 1)."""
    import torch
    import torch.distributed as dist

    import paper_1701_04733_b200 as bt
    from paper_1701_04733_b200.graphs import instance_seed, random_graph_matrix

    n = args.n or (32768 if args.workload == "fw" else 512)
    dtype = torch.int32 if args.workload == "fw" else torch.float32
    adj = random_graph_matrix(n, 0.5, (1, 100), instance_seed(1, n), dtype=dtype, device=dev)
    solver = bt.floyd_warshall if args.workload == "fw" else bt.apsp_by_squaring
    if args.workload == "apsp" and world > 1:
        # config C4: row-sharded squaring; the all-gather is fused into the
        # GEMM epilogue (peer stores into symmetric memory), NCCL fallback
        from paper_1701_04733_b200.sharded import apsp_by_squaring_distributed as solver  # noqa: F811
    elif args.workload == "fw" and world > 1:
        # row-sharded blocked FW; the pivot panel is stored into the peers by the owner's kernels
        from paper_1701_04733_b200.sharded import floyd_warshall_distributed as solver  # noqa: F811
    for _ in range(max(1, min(args.warmup, 3))):
        rep = solver(adj)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t = time.perf_counter()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.steps):
        rep = solver(adj)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    mults = rep.multiplications_performed
    pairs = float(n) ** 3 * (1 if args.workload == "fw" else mults)
    res = {"metric": f"APSP time n={n}", "value": round(ms / 1e3, 4), "unit": "s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": False,
           "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
           "dtype": "i32" if dtype == torch.int32 else "f32",
           "data": "synthetic",
           "config": {"workload": f"{args.workload}_n{n}", "graph": "random_graph p=0.5 weights 1..100",
                      "multiplications": mults, "negative_cycle": rep.negative_cycle,
                      "gpairs_per_s": round(pairs / (ms * 1e-3) / 1e9, 1)}}
    if args.workload == "apsp" and world > 1:
        res["config"]["exchange"] = os.environ.get("BTAS_EXCHANGE", "auto")
    # roofline: the add-min pairs of the whole solve against the live
    # ceiling of the s16x2 mix the integer-valued instances run on
    from paper_1701_04733_b200 import _lib

    probe = _lib.probe_ceiling(2)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    peak = probe["pairs_per_clk_sm"] * nsm * probe["sm_mhz"] * 1e6 / 1e12 * world
    ach = pairs / (ms * 1e-3) / 1e12
    res["roofline"] = {"bound": "alu", "achieved": round(ach, 3), "peak": round(peak, 3), "unit": "Tpair/s",
                       "frac": round(ach / peak, 4), "traffic": None,
                       "peak_source": "btas_probe_ceiling(s16x2) x SMs x probe clock x GPUs",
                       "work": "n^3 pairs (FW) / multiplications x n^3 (squaring), whole solve"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res["cpu_baseline"] = apsp_cpu_baseline(args.workload, n)
    if rank == 0:
        print(json.dumps(res), flush=True)
    return 0


def apsp_cpu_baseline(workload, n):
    """The reference's CPU algorithm on the host (oracle restatement, NumPy):
    C1 squaring in full; FW as a few k-rounds of the n' <= 4096 leading
    sub-instance (the reference round: d = min(d, d[:, k] (+) d[k, :])),
    extrapolated as n'^2 per round x n rounds x (n / n')^2."""
    import numpy as np

    from oracle import tropical as ot
    from paper_1701_04733_b200.graphs import dense_rows, instance_seed

    cores = len(os.sched_getaffinity(0))
    if workload == "apsp" and n <= 2048:
        sym = np.concatenate([blk for _, blk in dense_rows(n, 0.5, (1, 100), instance_seed(1, n))])
        ot.apsp_by_squaring(sym[:64, :64], "f32", True)  # warm-up
        t = time.perf_counter()
        ot.apsp_by_squaring(sym, "f32", True)
        secs = time.perf_counter() - t
        return {"value": round(secs, 4), "unit": "s", "cores": cores, "kind": "port",
                "sample": f"the full n={n} instance, NumPy restatement of apsp_by_squaring (threaded products)"}
    sub = min(n, 4096)
    rows = [blk for r0, blk in dense_rows(n, 0.5, (1, 100), instance_seed(1, n), chunk_rows=1024) if r0 < sub]
    d = np.ascontiguousarray(np.concatenate(rows)[:sub, :sub])
    np.fill_diagonal(d, np.minimum(np.diagonal(d), 0.0))
    rounds = 4
    t = time.perf_counter()
    for k in range(rounds):
        np.minimum(d, np.add.outer(d[:, k], d[k, :]), out=d)
    per_round = (time.perf_counter() - t) / rounds
    secs = per_round * (n / sub) ** 2 * n
    return {"value": round(secs, 1), "unit": "s", "cores": 1, "kind": "port",
            "sample": f"{rounds} reference FW rounds on the leading {sub}x{sub} block ({per_round:.3f} s/round), "
                      f"extrapolated x (n/{sub})^2 per round x n rounds"}


def hbm_arm(args, rank, world, dev):
    """Config C5: max-plus batched matvec / elementwise ⊕ at n = 65536 (f32,
    integers in [-1000, 1000], 10 % Infinity), HBM-bound: GB/s vs the
    measured copy bandwidth of MEASURED_PEAKS.json."""
    import torch

    import paper_1701_04733_b200 as bt
    from paper_1701_04733_b200 import matrix as bm

    n = args.n or 65536
    MAX = bt.SemiringKind.MAX_PLUS
    g = torch.Generator(device=dev)
    g.manual_seed(0xC5)

    def make(rows, cols):
        sym = torch.randint(-1000, 1001, (rows, cols), generator=g, device=dev, dtype=torch.int32).to(torch.float32)
        sym[torch.rand((rows, cols), generator=g, device=dev) < 0.10] = math.inf
        return bt.TropicalMatrix(MAX, sym, dtype=torch.float32, device=dev)

    A = make(n, n)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    if args.workload == "matvec":
        V = make(args.batch, n)
        fn = lambda: bt.matvec_batched(A, V)  # noqa: E731
        nbytes = (n * n + args.batch * n + args.batch * n) * 4
        wl = f"maxplus_matvec_n{n}_b{args.batch}_f32"
    else:
        B = make(n, n)
        fn = lambda: bt.ew_add(A, B)  # noqa: E731
        nbytes = 3 * n * n * 4
        wl = f"maxplus_ewadd_n{n}_f32"
    for _ in range(max(3, args.warmup)):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(int(dev.index)) as clocks:
        s.record()
        for _ in range(args.steps):
            fn()
        e.record()
        torch.cuda.synchronize()
    ms = s.elapsed_time(e) / args.steps
    gbs = nbytes / (ms * 1e-3) / 1e9
    res = {"metric": f"{wl} GB/s", "value": round(gbs, 1), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
           "warmup": max(3, args.warmup), "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": {"workload": wl, "n": n, "bytes_per_step": nbytes, "operands": "integers in [-1000,1000], 10% Inf",
                      "l2": "matrix 17 GB >> L2"},
           "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm, "unit": "GB/s",
                        "frac": round(gbs / hbm, 4), "traffic": None,
                        "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, read+write)"},
           "clocks": clocks.summary()}
    if rank == 0:
        print(json.dumps(res), flush=True)
    return 0


def graph_arm(args, rank, world, dev):
    """On-device instance generation: the C3 instance
    graph_to_matrix(random_graph(n, 0.5, (1, 100), instance_seed(1, n))) as
    int32 storage, through the public random_graph_matrix (presence, draw and
    fill kernels plus two 8-byte host reads).  HBM-bound on the matrix write
    and the draw array round trip; the host restatement (numpy PCG64,
    dense_rows) is timed beside it on a row sample."""
    import torch

    from paper_1701_04733_b200.graphs import dense_rows, instance_seed, random_graph_matrix

    n = args.n or 32768
    seed = instance_seed(1, n)
    fn = lambda: random_graph_matrix(n, 0.5, (1, 100), seed, dtype=torch.int32, device=dev)  # noqa: E731
    for _ in range(max(3, args.warmup)):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(int(dev.index)) as clocks:
        s.record()
        for _ in range(args.steps):
            m = fn()
        e.record()
        torch.cuda.synchronize()
    ms = s.elapsed_time(e) / args.steps
    edges = int((m.data < (1 << 28)).sum().item()) - n
    nbytes = n * n * 4 + edges * 4 * 2  # matrix write + draw array write and read
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    gbs = nbytes / (ms * 1e-3) / 1e9
    res = {"metric": f"instance generation n={n} G entries/s", "value": round(n * n / (ms * 1e-3) / 1e9, 2),
           "unit": "G entries/s", "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
           "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "i32", "data": "synthetic",
           "config": {"workload": f"random_graph_n{n}_i32", "graph": "random_graph p=0.5 weights 1..100",
                      "edges": edges, "bytes_per_step": nbytes, "l2": "matrix >> L2"},
           "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm, "unit": "GB/s",
                        "frac": round(gbs / hbm, 4), "traffic": None,
                        "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, read+write)",
                        "note": "also ALU-bound: 2.5 n^2 PCG64 128-bit steps per instance"},
           "clocks": clocks.summary()}
    if rank == 0 and world == 1:
        rows = 256
        t = time.perf_counter()
        for _ in dense_rows(n, 0.5, (1, 100), seed, chunk_rows=rows):
            break
        cpu_s = (time.perf_counter() - t) * n / rows
        res["cpu_baseline"] = {"value": round(n * n / cpu_s / 1e9, 4), "unit": "G entries/s", "cores": 1,
                               "kind": "port", "sample": f"first {rows} rows of the instance via dense_rows "
                               "(numpy PCG64 + scatter), extrapolated to n rows"}
    if rank == 0:
        print(json.dumps(res), flush=True)
    return 0


def reference_arm(args, rank, world):
    """The reference's own CPU algorithm (NumPy port of btas.matmul, every
    host thread) on a bounded sample of the same workload; rank 0 only."""
    if rank != 0:
        return 0
    import numpy as np

    from oracle import tropical as ot

    n = args.n or 16384
    rng = np.random.default_rng(0xB2000001)
    rows = cpu_sample_rows()
    xs = rng.integers(-1000, 1001, (rows, n)).astype(np.float64)
    xs[rng.random((rows, n)) < 0.25] = math.inf
    ys = rng.integers(-1000, 1001, (n, n)).astype(np.float64)
    ys[rng.random((n, n)) < 0.25] = math.inf
    xo, yo = ot.orient(ot.MIN, xs), ot.orient(ot.MIN, ys)
    cores = len(os.sched_getaffinity(0))
    times = []
    for i in range(args.warmup + args.steps):
        t = time.perf_counter()
        ot.matmul(xo, yo, ot.MIN, "i32", True, tile_rows=4, tile_cols=128, workers=cores)
        if i >= args.warmup:
            times.append(time.perf_counter() - t)
    pairs = rows * n * n
    value = pairs / statistics.median(times) / 1e9
    res = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(statistics.median(times) * 1e3, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "i32", "data": "synthetic", "impl": "reference",
        "config": {"workload": f"minplus_gemm_n{n}_i32", "n": n,
                   "sample": f"{rows} rows x {n} x {n} per step", "operands": "uniform integers in [-1000,1000]",
                   "infinity_fraction": 0.25},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{rows} rows x {n} x {n} per step (NumPy restatement of btas.matmul, "
                                   f"thread pool of {cores})"},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(res), flush=True)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
