#!/usr/bin/env python3
"""Benchmark of the tropical hot path on B200 (driver contract: one JSON line).

Default workload (BASELINE.json configs[1]): min-plus GEMM, n = 16384, int32
storage ("DPX"), operands uniform integers in [-1000, 1000] with 25 % Infinity
(the C2 recipe of SURVEY §8(d)).  One step = one C = A ⊗ B through the
product path (btas_gemm: screen, packing, GEMM kernel) with A, B resident in
HBM.  Metric: G(add,min)/s = n^3 / step time / 1e9.  The same line carries
``apsp_c4``: the n = 65536 repeated-squaring APSP (configs[3]) timed on every
rank, with its own roofline, clocks, e2e, CPU baseline and parity record.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                    [--workload gemm|gemm_f32|gemm_f32_real|fw|apsp|matvec|ewadd|graph] [--n N]

``--gpus N`` (N > 1) without a torchrun environment re-launches this script
under ``torch.distributed.run`` with N ranks (one per GPU, 127.0.0.1).  Under
torchrun every rank runs its own independent GEMM of the same size (the GEMM
shards into independent output blocks; no data-path collective: weak
scaling) and the C4 solve is row-sharded over the ranks (all-gather fused
into the GEMM epilogue); elapsed times are the max over ranks.

Keys beyond the base contract:
  roofline      the GEMM kernel's achieved pair rate (CUDA events around the
                kernel launches, on the launching stream) vs the live ceiling
                of its instruction mix (btas_probe_ceiling: pairs/clk/SM x SMs
                x the SM clock sampled during the timed region)
  cpu_baseline  the STOCK reference (btas.matmul, byte-compiled into
                oracle/_ref by oracle/ref_build.py) timed on this host's cores
                on a sampled row block of the same operands
  parity        byte comparison of the GPU result with that reference block
                (and, per variant / for C4, with the C oracle)
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
WORKLOADS = ["gemm", "gemm_f32", "gemm_f32_real", "fw", "apsp", "matvec", "ewadd", "graph", "verify", "paths"]


def parse(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[1])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="gemm", choices=WORKLOADS)
    ap.add_argument("--batch", type=int, default=1, help="vectors per matvec (config C5: 1, 2, 4, 8)")
    ap.add_argument("--n", type=int, default=0, help="problem size (default per workload)")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the byte comparisons against the reference/oracle")
    ap.add_argument("--no-apsp", action="store_true", help="skip the APSP C4 measurement of the default run")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the C1 / C3 / C5 measurements of the default run")
    ap.add_argument("--apsp-n", type=int, default=65536, help="APSP C4 size inside the default run")
    return ap.parse_args(argv)


# ---------------------------------------------------------------------------
# --gpus N: self-launch under torchrun when not already inside one
# ---------------------------------------------------------------------------
def _free_port() -> int:
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_command(argv, gpus: int, env) -> "list[str] | None":
    """The torchrun command that runs this script on ``gpus`` ranks, or None
    when no relaunch is needed (one GPU, or already a torchrun rank)."""
    if gpus <= 1 or "WORLD_SIZE" in env:
        return None
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
            *argv]


# ---------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------
class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int, period_ms: int = 100):
        self.gpu = gpu_index
        self.period = period_ms
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", str(self.period)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
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
        sm, mx, power, reasons = [], None, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
                power.append(float(parts[3]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    return json.loads(p.read_text()) if p.exists() else {}


def _hbm_peak():
    pk = _peaks()
    if "hbm_gbs" in pk:
        return float(pk["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, read+write)"
    return 6650.0, "B200_PROFILING.md fallback (MEASURED_PEAKS.json absent)"


# ---------------------------------------------------------------------------
# checker plumbing (test infrastructure: the stock reference and the oracle)
# ---------------------------------------------------------------------------
def _checks():
    """The checker (oracle/checks.py), imported only by the parity legs."""
    from oracle import checks

    return checks


def stock_reference():
    """The unmodified reference package (``btas``), byte-compiled into
    oracle/_ref by oracle/ref_build.py; its sources when run in the build
    container; None when neither exists."""
    try:
        from oracle import ref_build

        if ref_build.available():
            return ref_build.load()
        from oracle import ref_import

        if ref_import.available():
            return ref_import.load_reference()
    except ImportError:
        pass
    return None


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


def cpu_sample_rows():
    cores = len(os.sched_getaffinity(0))
    return int(min(128, max(8, 4 * cores)))


def reference_gemm_block(x_rows_sym, y_sym, kind_min=True):
    """The stock reference's btas.matmul on a row block (construction
    excluded, one untimed warm-up row, TileSpec(32, 32, all cores) — the best
    tile of SURVEY §8(d)'s sweep).  Returns (oriented float64 result,
    G pairs/s, seconds, cores, kind)."""
    cores = len(os.sched_getaffinity(0))
    btas = stock_reference()
    if btas is None:  # no compiled reference: the NumPy port of the same algorithm
        from oracle import tropical as ot

        k = ot.MIN if kind_min else ot.MAX
        xo, yo = ot.orient(k, x_rows_sym), ot.orient(k, y_sym)
        ot.matmul(xo[:1], yo, k, "f64", True, tile_rows=32, tile_cols=32, workers=cores)
        t = time.perf_counter()
        out, _ = ot.matmul(xo, yo, k, "f64", True, tile_rows=32, tile_cols=32, workers=cores)
        dt = time.perf_counter() - t
        return out, x_rows_sym.shape[0] * y_sym.size / dt / 1e9, dt, cores, "port"
    kind = btas.SemiringKind.MIN_PLUS if kind_min else btas.SemiringKind.MAX_PLUS
    Y = btas.TropicalMatrix(kind, y_sym)
    X = btas.TropicalMatrix(kind, x_rows_sym)
    tiles = btas.TileSpec(32, 32, cores)
    btas.matmul(btas.TropicalMatrix(kind, x_rows_sym[:1]), Y, tiles=tiles)  # warm-up (pool, pages)
    t = time.perf_counter()
    Z = btas.matmul(X, Y, tiles=tiles)
    dt = time.perf_counter() - t
    return Z.data, x_rows_sym.shape[0] * y_sym.size / dt / 1e9, dt, cores, "reference"


# ---------------------------------------------------------------------------
def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    cmd = relaunch_command(argv, args.gpus, os.environ)
    if cmd is not None:
        return subprocess.call(cmd)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, rank, world)

    import torch
    import torch.distributed as dist

    if local >= torch.cuda.device_count():
        raise SystemExit(f"bench.py: rank {rank} needs GPU {local}, but only {torch.cuda.device_count()} visible")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    arm = {"fw": apsp_arm, "apsp": apsp_arm, "matvec": hbm_arm, "ewadd": hbm_arm, "graph": graph_arm,
           "verify": verify_arm, "paths": paths_arm}.get(args.workload)
    if arm is not None:
        res = arm(args, rank, world, dev)
        if rank == 0:
            print(json.dumps(res), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return 0

    import paper_1701_04733_b200 as bt
    from paper_1701_04733_b200 import _lib
    from paper_1701_04733_b200 import matrix as bm

    n = args.n or 16384
    dtype, real, wl = {
        "gemm": (torch.int32, False, f"minplus_gemm_n{n}_i32"),
        "gemm_f32": (torch.float32, False, f"minplus_gemm_n{n}_f32_integer"),
        "gemm_f32_real": (torch.float32, True, f"minplus_gemm_n{n}_f32_real"),
    }[args.workload]

    # ------------------------------------------------------------- timed run
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
    if traffic is not None:
        roofline["traffic_note"] = ("dram bytes per launch (ncu --set full); above the compulsory 2-3 GB because "
                                    "L2 serves ~90 % of the 128 GB of tile loads — HBM runs at ~2 % of peak")

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
        result["variants"] = variants(n, dev, rank, check=not args.no_parity)

    # ------------------------------------------------------------- one product row-sharded over the ranks
    if world > 1 and args.workload == "gemm":
        try:
            result["gemm_row_sharded"] = gemm_row_sharded(args, n, dtype, real, world, dev)
        except Exception as exc:  # report, keep the line
            result["gemm_row_sharded"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    # ------------------------------------------------------------- stock reference on a row block (rank 0)
    # cpu_baseline (N = 1) and parity: the same operands, the reference's
    # btas.matmul on the first rows, byte-compared with the GPU's rows.
    if rank == 0 and not (args.no_cpu_baseline and args.no_parity):
        rows = cpu_sample_rows()
        xh = xs[:rows].double().cpu().numpy()
        yh = ys.double().cpu().numpy()
        ref, v, secs, cores, kind = reference_gemm_block(xh, yh)
        if world == 1 and not args.no_cpu_baseline:
            result["cpu_baseline"] = {
                "value": round(v, 4), "unit": UNIT, "cores": cores, "kind": kind,
                "sample": f"{rows} rows x {n} x {n} ({rows * n * n:.3g} pairs, {secs:.1f} s) of the same operands; "
                          + (f"stock btas.matmul(X[:{rows}], Y, tiles=TileSpec(32, 32, {cores})) (byte-compiled "
                             "oracle/_ref)" if kind == "reference" else
                             f"NumPy restatement of btas.matmul, 32x32 tiles on {cores} threads")
                          + ", float64 as the reference stores it, construction excluded",
            }
        if not args.no_parity:
            got = _checks().storage_to_f64(out[:rows]).cpu().numpy()
            result["parity"] = {"rows": rows, "cols": n, "mismatches": _checks().mismatches(got, ref),
                                "against": ("stock btas.matmul" if kind == "reference" else "NumPy port of btas.matmul")
                                + " on the same operands"}
        del yh
    result["_ref_gpairs"] = None  # filled below for C4's extrapolated CPU time
    if "cpu_baseline" in result:
        result["_ref_gpairs"] = result["cpu_baseline"]["value"]

    # ------------------------------------------------------------- the other BASELINE configs + C4
    # Every config of BASELINE.json is measured inside the default run, each
    # as a sub-line with its own roofline, clocks, e2e, cpu_baseline and
    # parity: C1 (n=512 squaring), C3 (n=32768 FW), C5 (n=65536 max-plus
    # matvec with 1 and 8 vectors, elementwise ⊕) and C4 (n=65536 squaring,
    # row-sharded over the ranks under torchrun).  A watchdog keeps the GEMM
    # line if anything stalls.
    if args.workload == "gemm" and not (args.no_apsp and args.no_configs):
        del x, y, out, xs, ys
        torch.cuda.empty_cache()

        def give_up():  # a stuck exchange must not cost the GEMM line
            result.setdefault("apsp_c4", {"error": f"timed out after {APSP_WATCHDOG_S} s"})
            result.pop("_ref_gpairs", None)
            if rank == 0:
                print(json.dumps(result), flush=True)
            os._exit(0)

        timer = threading.Timer(APSP_WATCHDOG_S, give_up)
        timer.daemon = True
        timer.start()
        try:
            if not args.no_configs:
                result["configs"] = {}
                subs = (("c1_apsp_n512", apsp_arm, dict(workload="apsp", n=512)),
                        ("c3_fw_n32768", apsp_arm, dict(workload="fw", n=32768, steps=3)),
                        ("c5_matvec_n65536_b1", hbm_arm, dict(workload="matvec", n=65536, batch=1)),
                        ("c5_matvec_n65536_b8", hbm_arm, dict(workload="matvec", n=65536, batch=8)),
                        # e2e of the 34 GB elementwise pair is PCIe-bound for seconds: its own arm has it
                        ("c5_ewadd_n65536", hbm_arm, dict(workload="ewadd", n=65536, no_e2e=True)))
                for key, arm, kw in subs:
                    try:
                        result["configs"][key] = arm(sub_args(args, **kw), rank, world, dev)
                    except Exception as exc:  # report, keep the rest
                        result["configs"][key] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
                    torch.cuda.empty_cache()
            if not args.no_apsp:
                try:
                    result["apsp_c4"] = apsp_c4(args, rank, world, dev, result.get("_ref_gpairs"))
                except Exception as exc:  # report, keep the GEMM line
                    result["apsp_c4"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        finally:
            timer.cancel()
    result.pop("_ref_gpairs", None)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


APSP_WATCHDOG_S = 1500


def sub_args(args, **kw):
    """A copy of the command-line namespace for one sub-measurement."""
    ns = argparse.Namespace(**vars(args))
    ns.steps = kw.pop("steps", args.steps)
    for k, v in kw.items():
        setattr(ns, k, v)
    return ns


def _max_over_ranks(v: float, world: int, dev) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _s16_ceiling(dev, sm_mhz=None):
    """Live ceiling of the s16x2 add-min mix the integer instances run on."""
    import torch

    from paper_1701_04733_b200 import _lib

    probe = _lib.probe_ceiling(2)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    mhz = sm_mhz or probe["sm_mhz"]
    return probe["pairs_per_clk_sm"] * nsm * mhz * 1e6 / 1e12, probe["pairs_per_clk_sm"], mhz


def gemm_row_sharded(args, n, dtype, real, world, dev):
    """SURVEY §8(e) GEMM row: ONE n x n product (the same operands on every
    rank) split by output rows over the ranks (matmul_distributed: B
    replicated, the all-gather fused into the GEMM epilogue as peer stores),
    strong scaling; every rank ends with the whole product, compared bytewise
    with its own single-GPU product."""
    import torch
    import torch.distributed as dist

    import paper_1701_04733_b200 as bt
    from paper_1701_04733_b200.sharded import matmul_distributed

    x, _ = gemm_inputs(n, dtype, dev, 0xB2000001, real)
    y, _ = gemm_inputs(n, dtype, dev, 0xB2000002, real)
    out = bt.matmul(x, y).data
    prod = matmul_distributed(x, y)  # warm-up (symmetric-memory rendezvous)
    torch.cuda.synchronize()
    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = max(1, min(args.steps, 5))
    s.record()
    for _ in range(steps):
        prod = matmul_distributed(x, y)
    e.record()
    torch.cuda.synchronize()
    ms = _max_over_ranks(s.elapsed_time(e) / steps, world, dev)
    same = bool(torch.equal(prod.data, out))  # this rank's own single-GPU product
    ok = torch.tensor([1 if same else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    return {"metric": f"row-sharded tropical GEMM G(add,min)/s at n={n}", "value": round(float(n) ** 3 /
            (ms * 1e-3) / 1e9, 1), "unit": UNIT, "n_gpus": world, "steps": steps, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "strong",
            "exchange": os.environ.get("BTAS_EXCHANGE", "auto"),
            "parity": {"equal_to_single_gpu_product_on_every_rank": bool(int(ok.item()))}}


def distance_checksum(d) -> int:
    """Sum of the finite distances (Infinity -> -1) mod 2^61: identical for
    every GPU count and for the e2e solve."""
    import torch

    checksum = 0
    for r0 in range(0, d.shape[0], 4096):
        blk = d[r0:r0 + 4096]
        blk = torch.where(torch.isfinite(blk), blk, torch.full_like(blk, -1)).to(torch.int64)
        checksum = (checksum + int(blk.sum().item())) % (1 << 61)
    return checksum


def apsp_c4(args, rank, world, dev, ref_gpairs=None):
    """BASELINE config C4 inside the default run: repeated-squaring APSP of
    the n = 65536 instance graph_to_matrix(random_graph(n, 0.5, (1, 100),
    instance_seed(1, n))) in fp32, on 1 GPU or row-sharded over the ranks
    (all-gather fused into the GEMM epilogue over symmetric memory, NCCL
    fallback).  One timed solve after a small warm-up solve; device time,
    max over ranks; then the same solve end to end through the public API
    from pinned host memory, and (rank 0) the parity record."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1701_04733_b200 as bt
    from paper_1701_04733_b200.graphs import instance_seed, random_graph_matrix

    n = args.apsp_n
    if world > 1:
        from paper_1701_04733_b200.sharded import apsp_by_squaring_distributed as solver
    else:
        solver = bt.apsp_by_squaring
    solver(random_graph_matrix(2048, 0.5, (1, 100), instance_seed(1, 2048), dtype=torch.float32, device=dev))
    seed = instance_seed(1, n)
    adj = random_graph_matrix(n, 0.5, (1, 100), seed, dtype=torch.float32, device=dev)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clocks:
        s.record()
        rep = solver(adj)
        e.record()
        torch.cuda.synchronize()
    ms = _max_over_ranks(s.elapsed_time(e), world, dev)
    clk = clocks.summary()
    mults = rep.multiplications_performed
    pairs = float(n) ** 3 * mults
    d = rep.distances.dist.data
    checksum = distance_checksum(d)
    peak1, ppc, mhz = _s16_ceiling(dev, clk["sm_mhz"])
    ach = pairs / (ms * 1e-3) / 1e12
    out = {"metric": f"APSP time n={n}", "value": round(ms / 1e3, 3), "unit": "s", "higher_is_better": False,
           "n_gpus": world, "scaling": "strong", "dtype": "f32", "data": "synthetic",
           "config": {"workload": f"apsp_squaring_n{n}_f32", "graph": "random_graph p=0.5 weights 1..100",
                      "instance_seed": "instance_seed(1, n)", "l2": "matrix 16 GiB >> L2"},
           "multiplications": mults, "negative_cycle": rep.negative_cycle,
           "distance_checksum": checksum,
           "tpairs_per_s": round(ach, 2),
           "roofline": {"bound": "alu", "achieved": round(ach, 3), "peak": round(peak1 * world, 3), "unit": "Tpair/s",
                        "frac": round(ach / (peak1 * world), 4), "traffic": None,
                        "work": "multiplications x n^3 add-min pairs (the uncounted probe is not run: fixpoint)",
                        "peak_source": f"btas_probe_ceiling(s16x2) {ppc:.1f} pairs/clk/SM x SMs x {mhz} MHz "
                                       f"(median SM clock of the solve) x {world} GPU(s)"},
           "clocks": clk}
    if world > 1:
        out["exchange"] = os.environ.get("BTAS_EXCHANGE", "auto")
    if ref_gpairs:
        cpu_s = pairs / (ref_gpairs * 1e9)
        out["cpu_baseline"] = {"value": round(cpu_s, 1), "unit": "s", "cores": len(os.sched_getaffinity(0)),
                               "kind": "reference", "extrapolated": True,
                               "sample": f"multiplications x n^3 / the stock btas.matmul rate measured in this run "
                                         f"on the C2 row block ({ref_gpairs} G pairs/s); the float64 n=65536 "
                                         "matrix (34 GB per operand) does not fit the reference's host path"}

    # ------------------------------------------------------------- e2e through the public API
    if not args.no_e2e:
        try:
            hadj = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
            for r0 in range(0, n, 4096):  # symbolic form: +inf absent
                hadj[r0 : r0 + 4096].copy_(adj.data[r0 : r0 + 4096])
            hout = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
            del rep, d
            torch.cuda.empty_cache()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            A = bt.TropicalMatrix(bt.SemiringKind.MIN_PLUS, hadj, dtype=torch.float32, device=dev)
            rep = solver(A)
            hout.copy_(rep.distances.dist.data, non_blocking=True)
            torch.cuda.synchronize()
            e2e_s = _max_over_ranks(time.perf_counter() - t0, world, dev)
            del A
            out["e2e"] = {"value": round(e2e_s, 3), "unit": "s", "h2d_bytes_per_step": n * n * 4,
                          "d2h_bytes_per_step": n * n * 4,
                          "path": "pinned host f32 adjacency -> TropicalMatrix (H2D + validation/ingest) -> "
                                  f"{'apsp_by_squaring_distributed' if world > 1 else 'apsp_by_squaring'} -> "
                                  "distances D2H into pinned memory (wall clock, one solve)"}
            d = rep.distances.dist.data
            out["e2e"]["same_checksum_as_timed_solve"] = distance_checksum(d) == checksum
            out["e2e"]["host_rows_equal_device"] = bool(
                np.array_equal(hout[-64:].numpy().view(np.int32), d[-64:].cpu().numpy().view(np.int32)))
            del hadj, hout
        except (RuntimeError, MemoryError) as exc:
            out["e2e"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
            d = rep.distances.dist.data

    # ------------------------------------------------------------- parity (rank 0)
    if rank == 0 and not args.no_parity:
        try:
            rng = np.random.default_rng(0xC4)
            sample = sorted({0, n - 1, *rng.choice(n, 14, replace=False).tolist()})
            out["parity"] = _checks().closure_rows_parity(adj.data, d, sample, gen=(n, 0.5, (1, 100), seed))
        except Exception as exc:  # the measurement stands; the failed check is reported
            out["parity"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    if world > 1:
        dist.barrier()
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


def variants(n, dev, rank, check=True):
    """The other kernel paths on the same size (fewer steps); each checked
    on 8 sampled rows against the C oracle (storage-aware restatement of
    btas.matmul)."""
    import numpy as np
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
        "f64_real_valued": (torch.float64, True, 1000),
    }
    storage = {torch.float32: "f32", torch.int32: "i32", torch.float64: "f64"}
    for name, (dtype, real, rng) in cases.items():
        g = torch.Generator(device=dev)
        g.manual_seed(0xB2000002 + rank)
        mats, syms = [], []
        for _ in range(2):
            if real:
                sym = torch.rand((n, n), generator=g, device=dev, dtype=torch.float64) * 2000.0 - 1000.0
                if dtype == torch.float32:
                    sym = sym.to(torch.float32)
            else:
                sym = torch.randint(-rng, rng + 1, (n, n), generator=g, device=dev, dtype=torch.int32).to(torch.float32)
            sym[torch.rand((n, n), generator=g, device=dev) < 0.25] = math.inf
            mats.append(bt.TropicalMatrix(bt.SemiringKind.MIN_PLUS, sym, dtype=dtype, device=dev))
            syms.append(sym)
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
        mix = {"s16x2": 2, "i32f64": 1, "fast64": 3}.get(path, 1 if dtype == torch.int32 else 0)
        try:
            probe = _lib.probe_ceiling(mix)
            nsm = torch.cuda.get_device_properties(dev).multi_processor_count
            peak = probe["pairs_per_clk_sm"] * nsm * probe["sm_mhz"] * 1e6 / 1e12
        except RuntimeError:  # no probe for this mix
            peak = None
        ach = float(n) ** 3 / (kms / kc * 1e-3) / 1e12
        out[name] = {"value": round(float(n) ** 3 / (ms * 1e-3) / 1e9, 1), "unit": UNIT, "kernel_path": path,
                     "kernel_tpairs": round(ach, 3), "peak_tpairs_probe_clock": round(peak, 3) if peak else None,
                     "frac": round(ach / peak, 4) if peak else None}
        if check:
            from oracle import native

            rows = 8
            xh = syms[0][:rows].double().cpu().numpy()
            yh = syms[1].double().cpu().numpy()
            want, _ = native.matmul(xh, yh, "minplus", storage[dtype], integer)
            got = _checks().storage_to_f64(o[:rows]).cpu().numpy()
            out[name]["parity"] = {"rows": rows, "mismatches": _checks().mismatches(got, want),
                                   "against": "oracle_gemm (C restatement of btas.matmul)"}
            del yh
        del x, y, o, mats, syms
        torch.cuda.empty_cache()
    return out


def apsp_arm(args, rank, world, dev):
    """FW (C3) / squaring (C1, C4) timing: 1 GPU, or row-sharded over the
    ranks (squaring: fused all-gather; FW: pivot-panel distribution)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1701_04733_b200 as bt
    from paper_1701_04733_b200.graphs import instance_seed, random_graph_matrix
    from paper_1701_04733_b200.matrix import _to_f64

    n = args.n or (32768 if args.workload == "fw" else 512)
    dtype = torch.int32 if args.workload == "fw" else torch.float32
    seed = instance_seed(1, n)
    adj = random_graph_matrix(n, 0.5, (1, 100), seed, dtype=dtype, device=dev)
    solver = bt.floyd_warshall if args.workload == "fw" else bt.apsp_by_squaring
    if args.workload == "apsp" and world > 1:
        from paper_1701_04733_b200.sharded import apsp_by_squaring_distributed as solver  # noqa: F811
    elif args.workload == "fw" and world > 1:
        from paper_1701_04733_b200.sharded import floyd_warshall_distributed as solver  # noqa: F811
    for _ in range(max(3, args.warmup)):
        rep = solver(adj)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = solver(adj)
    torch.cuda.synchronize()
    # small solves (C1: 0.2 ms) repeat until the timed region spans >= 1.5 s
    # so the clock sampler sees it; the same count on every rank
    steps = int(_max_over_ranks(max(args.steps, math.ceil(1.5 / max(time.perf_counter() - t0, 1e-5))), world, dev))
    if world > 1:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index, period_ms=50) as clocks:
        s.record()
        for _ in range(steps):
            rep = solver(adj)
        e.record()
        torch.cuda.synchronize()
    ms = _max_over_ranks(s.elapsed_time(e) / steps, world, dev)
    clk = clocks.summary()
    mults = rep.multiplications_performed
    pairs = float(n) ** 3 * (1 if args.workload == "fw" else mults)
    res = {"metric": f"APSP time n={n}", "value": round(ms / 1e3, 6), "unit": "s", "n_gpus": world,
           "steps": steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms, 3), "higher_is_better": False,
           "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
           "dtype": "i32" if dtype == torch.int32 else "f32",
           "data": "synthetic",
           "config": {"workload": f"{args.workload}_n{n}", "graph": "random_graph p=0.5 weights 1..100",
                      "instance_seed": "instance_seed(1, n)",
                      "multiplications": mults, "negative_cycle": rep.negative_cycle,
                      "gpairs_per_s": round(pairs / (ms * 1e-3) / 1e9, 1),
                      "l2": "matrix >> L2" if n * n * 4 > 126e6 else "matrix L2-resident (C1 is latency-bound)"},
           "clocks": clk, "gpu_launches": None}
    if world > 1:
        res["config"]["exchange"] = os.environ.get("BTAS_EXCHANGE", "auto")
    peak, ppc, mhz = _s16_ceiling(dev, clk["sm_mhz"])
    ach = pairs / (ms * 1e-3) / 1e12
    res["roofline"] = {"bound": "alu", "achieved": round(ach, 3), "peak": round(peak * world, 3), "unit": "Tpair/s",
                       "frac": round(ach / (peak * world), 4), "traffic": None,
                       "peak_source": f"btas_probe_ceiling(s16x2) {ppc:.1f} pairs/clk/SM x SMs x {mhz} MHz x GPUs",
                       "work": "n^3 pairs (FW) / multiplications x n^3 (squaring), whole solve"}
    # e2e: pinned host symbolic adjacency -> TropicalMatrix -> solve -> D2H
    if not args.no_e2e:
        hadj = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
        hadj.copy_(_to_f64(adj.data).to(torch.float32))  # symbolic min-plus form = oriented
        hout = torch.empty((n, n), dtype=dtype, pin_memory=True)
        k = max(1, min(args.steps, 3))

        def e2e_once():
            A = bt.TropicalMatrix(bt.SemiringKind.MIN_PLUS, hadj, dtype=dtype, device=dev)
            r = solver(A)
            hout.copy_(r.distances.dist.data, non_blocking=True)
            torch.cuda.synchronize()

        e2e_once()
        t0 = time.perf_counter()
        for _ in range(k):
            e2e_once()
        e2e_s = _max_over_ranks((time.perf_counter() - t0) / k, world, dev)
        res["e2e"] = {"value": round(e2e_s, 4), "unit": "s", "h2d_bytes_per_step": n * n * 4,
                      "d2h_bytes_per_step": n * n * 4,
                      "path": "pinned host f32 adjacency -> TropicalMatrix -> solver -> distances D2H (wall clock)"}
        del hadj, hout
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res["cpu_baseline"], ref_d = apsp_cpu_baseline(args.workload, n)
    else:
        ref_d = None
    if rank == 0 and not args.no_parity:
        d = rep.distances.dist.data
        if ref_d is not None:  # C1: the stock reference solved the whole instance
            want, want_mults = ref_d
            got = _checks().storage_to_f64(d).cpu().numpy()
            res["parity"] = {"rows": n, "cols": n, "mismatches": _checks().mismatches(got, want),
                             "multiplications_equal": want_mults == mults if args.workload == "apsp" else None,
                             "against": "btas.apsp_by_squaring (stock reference) on the same instance"}
        else:
            rng = np.random.default_rng(0xC3)
            sample = sorted({0, n - 1, *rng.choice(n, 14, replace=False).tolist()})
            res["parity"] = _checks().closure_rows_parity(adj.data, d, sample, gen=(n, 0.5, (1, 100), seed))
    return res


def apsp_cpu_baseline(workload, n):
    """The reference's CPU algorithm on the host: the stock
    btas.apsp_by_squaring on the full instance when it fits (C1), else FW as
    a few reference k-rounds on the leading n' <= 4096 block, extrapolated
    as n'^2 per round x n rounds x (n / n')^2.  Returns (record, (oriented
    float64 distances, multiplications) or None)."""
    import numpy as np

    from oracle import tropical as ot
    from paper_1701_04733_b200.graphs import dense_rows, instance_seed

    cores = len(os.sched_getaffinity(0))
    btas = stock_reference()
    if n <= 2048 and (workload == "apsp" or n <= 1024):
        sym = np.concatenate([blk for _, blk in dense_rows(n, 0.5, (1, 100), instance_seed(1, n))])
        if btas is not None:
            adj = btas.TropicalMatrix(btas.SemiringKind.MIN_PLUS, sym)
            btas.apsp_by_squaring(btas.TropicalMatrix(btas.SemiringKind.MIN_PLUS, sym[:64, :64]))  # warm-up
            solve = btas.floyd_warshall if workload == "fw" else btas.apsp_by_squaring
            times = []
            for _ in range(3):
                t = time.perf_counter()
                rep = solve(adj)
                times.append(time.perf_counter() - t)
            secs = statistics.median(times)
            ref = (rep.distances.dist.data, rep.multiplications_performed)
            kind, what = "reference", f"btas.{solve.__name__} (stock reference, default TileSpec), median of 3"
        else:
            t = time.perf_counter()
            d, _, mults, _ = ot.apsp_by_squaring(sym, "f32", True)
            secs = time.perf_counter() - t
            ref = None
            kind, what = "port", "NumPy restatement of apsp_by_squaring"
        return {"value": round(secs, 4), "unit": "s", "cores": cores, "kind": kind,
                "sample": f"the full n={n} instance, {what}"}, ref
    if workload == "fw" and btas is not None:
        # the stock reference's floyd_warshall (apsp.py:93-133: numpy rounds,
        # single-threaded like the reference) on a bounded instance, scaled by
        # its n^3 work
        m = 1024
        sym = np.concatenate([blk for _, blk in dense_rows(m, 0.5, (1, 100), instance_seed(1, m))])
        A = btas.TropicalMatrix(btas.SemiringKind.MIN_PLUS, sym)
        btas.floyd_warshall(btas.TropicalMatrix(btas.SemiringKind.MIN_PLUS, sym[:64, :64]))  # warm-up
        t = time.perf_counter()
        btas.floyd_warshall(A)
        secs = time.perf_counter() - t
        return {"value": round(secs * (n / m) ** 3, 1), "unit": "s", "cores": 1, "kind": "reference",
                "extrapolated": True,
                "sample": f"stock btas.floyd_warshall on the n={m} instance ({secs:.2f} s, numpy rounds on one "
                          f"core as the reference runs them), x (n/{m})^3"}, None
    sub = min(n, 4096)
    rows = [blk for r0, blk in dense_rows(n, 0.5, (1, 100), instance_seed(1, n), chunk_rows=1024) if r0 < sub]
    d = np.ascontiguousarray(np.concatenate(rows)[:sub, :sub])
    np.fill_diagonal(d, np.minimum(np.diagonal(d), 0.0))
    rounds = 4
    t = time.perf_counter()
    for k in range(rounds):  # the reference round (apsp.py:108-109)
        np.minimum(d, np.add.outer(d[:, k], d[k, :]), out=d)
    per_round = (time.perf_counter() - t) / rounds
    secs = per_round * (n / sub) ** 2 * n
    return {"value": round(secs, 1), "unit": "s", "cores": 1, "kind": "port", "extrapolated": True,
            "sample": f"{rounds} reference FW rounds (apsp.py:108-109, single-threaded like the reference) on the "
                      f"leading {sub}x{sub} block ({per_round:.3f} s/round), extrapolated x (n/{sub})^2 per round "
                      "x n rounds"}, None


def hbm_arm(args, rank, world, dev):
    """Config C5: max-plus batched matvec / elementwise ⊕ at n = 65536 (f32,
    integers in [-1000, 1000], 10 % Infinity), HBM-bound: GB/s vs the
    measured copy bandwidth of MEASURED_PEAKS.json.  The timed region is
    stretched to >= 1.5 s (more steps) so the clock sampler sees it."""
    import numpy as np
    import torch

    import paper_1701_04733_b200 as bt

    n = args.n or 65536
    MAX = bt.SemiringKind.MAX_PLUS
    g = torch.Generator(device=dev)
    g.manual_seed(0xC5)

    def make_sym(rows, cols):
        sym = torch.randint(-1000, 1001, (rows, cols), generator=g, device=dev, dtype=torch.int32).to(torch.float32)
        sym[torch.rand((rows, cols), generator=g, device=dev) < 0.10] = math.inf
        return sym

    a_sym = make_sym(n, n)
    A = bt.TropicalMatrix(MAX, a_sym, dtype=torch.float32, device=dev)
    hbm, hbm_src = _hbm_peak()
    if args.workload == "matvec":
        v_sym = make_sym(args.batch, n)
        V = bt.TropicalMatrix(MAX, v_sym, dtype=torch.float32, device=dev)
        fn = lambda: bt.matvec_batched(A, V)  # noqa: E731
        nbytes = (n * n + args.batch * n + args.batch * n) * 4
        wl = f"maxplus_matvec_n{n}_b{args.batch}_f32"
    else:
        b_sym = make_sym(n, n)
        B = bt.TropicalMatrix(MAX, b_sym, dtype=torch.float32, device=dev)
        fn = lambda: bt.ew_add(A, B)  # noqa: E731
        nbytes = 3 * n * n * 4
        wl = f"maxplus_ewadd_n{n}_f32"
    for _ in range(max(3, args.warmup)):
        res_t = fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    est = time.perf_counter() - t0
    steps = max(args.steps, int(math.ceil(1.5 / max(est, 1e-4))))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index, period_ms=50) as clocks:
        s.record()
        for _ in range(steps):
            res_t = fn()
        e.record()
        torch.cuda.synchronize()
    ms = _max_over_ranks(s.elapsed_time(e) / steps, world, dev)
    gbs = nbytes / (ms * 1e-3) / 1e9
    res = {"metric": f"{wl} GB/s", "value": round(gbs * world, 1), "unit": "GB/s", "n_gpus": world, "steps": steps,
           "warmup": max(3, args.warmup), "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": {"workload": wl, "n": n, "bytes_per_step": nbytes, "operands": "integers in [-1000,1000], 10% Inf",
                      "l2": "matrix 17 GB >> L2", "steps_note": "steps raised so the timed region is >= 1.5 s"},
           "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm, "unit": "GB/s",
                        "frac": round(gbs / hbm, 4), "traffic": None, "peak_source": hbm_src},
           "clocks": clocks.summary(), "gpu_launches": steps}
    if not args.no_e2e:  # the public API from pinned host memory (A stays resident for matvec: it is the operator)
        if args.workload == "matvec":
            hv = v_sym.cpu().pin_memory()
            hout = torch.empty((args.batch, n), dtype=torch.float32, pin_memory=True)

            def once():
                Vh = bt.TropicalMatrix(MAX, hv, dtype=torch.float32, device=dev)
                hout.copy_(bt.matvec_batched(A, Vh), non_blocking=True)
                torch.cuda.synchronize()

            h2d, d2h = args.batch * n * 4, args.batch * n * 4
            what = "pinned host vectors -> TropicalMatrix -> matvec_batched(A resident) -> D2H"
        else:
            ha, hb = a_sym.cpu().pin_memory(), b_sym.cpu().pin_memory()
            hout = torch.empty((n, n), dtype=torch.float32, pin_memory=True)

            def once():
                Ah = bt.TropicalMatrix(MAX, ha, dtype=torch.float32, device=dev)
                Bh = bt.TropicalMatrix(MAX, hb, dtype=torch.float32, device=dev)
                hout.copy_(bt.ew_add(Ah, Bh).data, non_blocking=True)
                torch.cuda.synchronize()

            h2d, d2h = 2 * n * n * 4, n * n * 4
            what = "pinned host operands -> TropicalMatrix x2 -> ew_add -> D2H (PCIe-bound)"
        once()
        k = 3
        t0 = time.perf_counter()
        for _ in range(k):
            once()
        es = _max_over_ranks((time.perf_counter() - t0) / k, world, dev)
        res["e2e"] = {"value": round(nbytes * world / es / 1e9, 1), "unit": "GB/s", "h2d_bytes_per_step": h2d,
                      "d2h_bytes_per_step": d2h, "ms_per_step": round(es * 1e3, 2), "path": what}
    if rank == 0 and not args.no_parity:  # 8 sampled rows against the oracle
        from oracle import tropical as ot

        rng = np.random.default_rng(0xC5)
        rows = sorted(rng.choice(n, 8, replace=False).tolist())
        a_rows = a_sym[rows].double().cpu().numpy()
        got_all = res_t if args.workload == "matvec" else res_t.data
        if args.workload == "matvec":
            vh = v_sym.double().cpu().numpy()
            bad = 0
            for b in range(args.batch):
                want, _ = ot.matvec(ot.orient(ot.MAX, a_rows), ot.orient(ot.MAX, vh[b]), ot.MAX, "f32", True)
                bad += _checks().mismatches(_checks().storage_to_f64(got_all[b, rows]).cpu().numpy(), want)
            what = "oracle.tropical.matvec (btas.matvec restated) on 8 sampled output rows x every vector"
        else:
            b_rows = b_sym[rows].double().cpu().numpy()
            want = ot.ew_add(ot.orient(ot.MAX, a_rows), ot.orient(ot.MAX, b_rows), ot.MAX)
            bad = _checks().mismatches(_checks().storage_to_f64(got_all[rows]).cpu().numpy(), want)
            what = "oracle.tropical.ew_add (btas.ew_add restated) on 8 sampled rows"
        res["parity"] = {"rows": rows, "mismatches": bad, "against": what}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res["cpu_baseline"] = hbm_cpu_baseline(args.workload, a_sym, v_sym if args.workload == "matvec" else b_sym,
                                               nbytes, n)
    return res


def hbm_cpu_baseline(workload, a_sym, other_sym, nbytes, n):
    """The stock reference (btas.matvec / btas.ew_add, float64) on a row
    sample of the same operands, extrapolated to the full matrix bytes of
    the device metric."""
    cores = len(os.sched_getaffinity(0))
    btas = stock_reference()
    rows = 512
    a = a_sym[:rows].double().cpu().numpy()
    MAX = btas.SemiringKind.MAX_PLUS if btas is not None else None
    if btas is None:
        return {"value": None, "unit": "GB/s", "cores": 1, "kind": "port", "sample": "compiled reference missing"}
    A = btas.TropicalMatrix(MAX, a)
    if workload == "matvec":
        vs = other_sym.double().cpu().numpy()
        V = [btas.TropicalVector(MAX, vs[b]) for b in range(vs.shape[0])]
        btas.matvec(A, V[0])
        t = time.perf_counter()
        for v in V:
            btas.matvec(A, v)
        dt = time.perf_counter() - t
        what = f"btas.matvec on the first {rows} rows x {len(V)} vector(s)"
    else:
        B = btas.TropicalMatrix(MAX, other_sym[:rows].double().cpu().numpy())
        btas.ew_add(A, B)
        t = time.perf_counter()
        btas.ew_add(A, B)
        dt = time.perf_counter() - t
        what = f"btas.ew_add on the first {rows} rows"
    full_s = dt * n / rows
    return {"value": round(nbytes / full_s / 1e9, 3), "unit": "GB/s", "cores": 1, "kind": "reference",
            "extrapolated": True,
            "sample": f"{what} (float64, single-threaded like the reference), extrapolated x n/{rows}; "
                      "GB/s over the same f32 algorithmic bytes as the device metric"}


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
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    steps = max(args.steps, int(math.ceil(1.5 / max(time.perf_counter() - t0, 1e-4))))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(int(dev.index), period_ms=50) as clocks:
        s.record()
        for _ in range(steps):
            m = fn()
        e.record()
        torch.cuda.synchronize()
    ms = _max_over_ranks(s.elapsed_time(e) / steps, world, dev)
    edges = int((m.data < (1 << 28)).sum().item()) - n
    nbytes = n * n * 4 + edges * 4 * 2  # matrix write + draw array write and read
    hbm, hbm_src = _hbm_peak()
    gbs = nbytes / (ms * 1e-3) / 1e9
    res = {"metric": f"instance generation n={n} G entries/s", "value": round(n * n * world / (ms * 1e-3) / 1e9, 2),
           "unit": "G entries/s", "n_gpus": world, "steps": steps, "warmup": max(3, args.warmup),
           "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "i32", "data": "synthetic",
           "config": {"workload": f"random_graph_n{n}_i32", "graph": "random_graph p=0.5 weights 1..100",
                      "edges": edges, "bytes_per_step": nbytes, "l2": "matrix >> L2"},
           "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm, "unit": "GB/s",
                        "frac": round(gbs / hbm, 4), "traffic": None, "peak_source": hbm_src,
                        "note": "also ALU-bound: 2.5 n^2 PCG64 128-bit steps per instance"},
           "clocks": clocks.summary(), "gpu_launches": steps * 4}
    if rank == 0 and not args.no_parity:
        from oracle import graphs as og

        bad = 0
        for r0 in (0, n // 2, n - 64):
            want = og.instance_rows(n, 0.5, (1, 100), seed, r0, r0 + 64)
            bad += _checks().mismatches(_checks().storage_to_f64(m.data[r0 : r0 + 64]).cpu().numpy(), want)
        res["parity"] = {"rows": "3 blocks of 64 (first, middle, last)", "mismatches": bad,
                         "against": "oracle.graphs.instance_rows (numpy PCG64 stream of random_graph)"}
    if rank == 0 and world == 1:
        rows = 256
        t = time.perf_counter()
        for _ in dense_rows(n, 0.5, (1, 100), seed, chunk_rows=rows):
            break
        cpu_s = (time.perf_counter() - t) * n / rows
        res["cpu_baseline"] = {"value": round(n * n / cpu_s / 1e9, 4), "unit": "G entries/s", "cores": 1,
                               "kind": "port", "extrapolated": True,
                               "sample": f"first {rows} rows of the instance via dense_rows "
                               "(numpy PCG64 + scatter), extrapolated to n rows"}
    return res


def verify_arm(args, rank, world, dev):
    """The fused on-GPU verifier (reference
    find_apsp_violation, apsp.py:181-210) on the C4 instance: squaring solve
    (untimed), then one timed find_apsp_violation — btas_verify_base plus two
    btas_gemm_verify products (2 n^3 add-min pairs, nothing stored)."""
    import torch

    import paper_1701_04733_b200 as bt
    from paper_1701_04733_b200.graphs import instance_seed, random_graph_matrix

    n = args.n or 65536
    small = random_graph_matrix(2048, 0.5, (1, 100), instance_seed(1, 2048), dtype=torch.float32, device=dev)
    assert bt.find_apsp_violation(small, bt.apsp_by_squaring(small).distances) is None  # warm-up
    adj = random_graph_matrix(n, 0.5, (1, 100), instance_seed(1, n), dtype=torch.float32, device=dev)
    dm = bt.apsp_by_squaring(adj).distances
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clocks:
        s.record()
        verdict = bt.find_apsp_violation(adj, dm)
        e.record()
        torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    clk = clocks.summary()
    pairs = 2.0 * float(n) ** 3
    peak, ppc, mhz = _s16_ceiling(dev, clk["sm_mhz"])
    ach = pairs / (ms * 1e-3) / 1e12
    # a broken copy: the first bad diagonal entry is named exactly
    bad = dm.dist.data.clone()
    bad[4321, 4321] = 1.0
    msg = bt.find_apsp_violation(adj, bt.DistanceMatrix(n, bt.TropicalMatrix._wrap(bt.SemiringKind.MIN_PLUS, bad,
                                                                                   True)))
    del bad
    res = {"metric": f"find_apsp_violation time n={n}", "value": round(ms / 1e3, 3), "unit": "s", "n_gpus": world,
           "steps": 1, "warmup": 1, "ms_per_step": round(ms, 1), "higher_is_better": False, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": {"workload": f"verify_squaring_n{n}_f32", "graph": "random_graph p=0.5 weights 1..100",
                      "checks": "diag, d <= I(+)A, d <= d(x)d, d == d(x)(I(+)A)"},
           "roofline": {"bound": "alu", "achieved": round(ach, 3), "peak": round(peak, 3), "unit": "Tpair/s",
                        "frac": round(ach / peak, 4), "traffic": None,
                        "work": "2 n^3 add-min pairs (the two verifier products)",
                        "peak_source": f"btas_probe_ceiling(s16x2) {ppc:.1f} pairs/clk/SM x SMs x {mhz} MHz"},
           "clocks": clk, "gpu_launches": 2 * 11 + 1,
           "parity": {"true_distances": verdict, "broken_diagonal": msg,
                      "expected_broken": "diagonal entry (4321,4321) is np.float64(1.0), expected 0"}}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        btas = stock_reference()
        if btas is not None:  # the reference verifier on a bounded instance, extrapolated by its n^3 work
            import numpy as np

            from paper_1701_04733_b200.graphs import dense_rows

            m = 768
            sym = np.concatenate([blk for _, blk in dense_rows(m, 0.5, (1, 100), instance_seed(1, m))])
            A = btas.TropicalMatrix(btas.SemiringKind.MIN_PLUS, sym)
            D = btas.apsp_by_squaring(A).distances
            t = time.perf_counter()
            assert btas.find_apsp_violation(A, D) is None
            secs = time.perf_counter() - t
            res["cpu_baseline"] = {"value": round(secs * (n / m) ** 3, 1), "unit": "s",
                                   "cores": len(os.sched_getaffinity(0)), "kind": "reference", "extrapolated": True,
                                   "sample": f"stock btas.find_apsp_violation on the n={m} instance ({secs:.2f} s), "
                                             f"x (n/{m})^3"}
    return res


def paths_arm(args, rank, world, dev):
    """Path reconstruction: the predecessor product
    btas_gemm_argmin (n^3 candidates, first argmin k per output) on the
    n = 16384 int32 instance after its Floyd-Warshall solve."""
    import torch

    import paper_1701_04733_b200 as bt
    from paper_1701_04733_b200 import _lib
    from paper_1701_04733_b200.graphs import instance_seed, random_graph_matrix

    n = args.n or 16384
    adj = random_graph_matrix(n, 0.5, (1, 100), instance_seed(1, n), dtype=torch.int32, device=dev)
    rep = bt.floyd_warshall(adj)
    for _ in range(max(1, args.warmup)):
        pred = bt.predecessors(adj, rep)
    torch.cuda.synchronize()
    steps = max(1, args.steps)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clocks:
        s.record()
        for _ in range(steps):
            pred = bt.predecessors(adj, rep)
        e.record()
        torch.cuda.synchronize()
    ms = s.elapsed_time(e) / steps
    clk = clocks.summary()
    probe = _lib.probe_ceiling(1)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    mhz = clk["sm_mhz"] or probe["sm_mhz"]
    peak = probe["pairs_per_clk_sm"] * nsm * mhz * 1e6 / 1e12
    ach = float(n) ** 3 / (ms * 1e-3) / 1e12
    unreachable = int((pred < 0).sum().item()) - n
    res = {"metric": f"predecessor product n={n} Tpair/s", "value": round(ach, 3), "unit": "Tpair/s",
           "n_gpus": world, "steps": steps, "warmup": max(1, args.warmup), "ms_per_step": round(ms, 2),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "i32", "data": "synthetic",
           "config": {"workload": f"predecessors_n{n}_i32", "graph": "random_graph p=0.5 weights 1..100",
                      "unreachable_pairs": unreachable},
           "roofline": {"bound": "alu", "achieved": round(ach, 3), "peak": round(peak, 3), "unit": "Tpair/s",
                        "frac": round(ach / peak, 4), "traffic": None,
                        "work": "n^3 candidates; small integer data: packed (value << 16 | k) keys, one "
                                "VIADDMNMX per candidate (else compare-and-select, ~3 ALU ops)",
                        "peak_source": "btas_probe_ceiling(i32 VIADDMNMX, 1 instruction per pair) x SMs x clock"},
           "clocks": clk, "gpu_launches": steps * 3}
    return res


def reference_arm(args, rank, world):
    """The stock reference's CPU path (btas.matmul, byte-compiled into
    oracle/_ref; the NumPy port only if that is missing) on every host core,
    on a bounded row sample of the same workload; rank 0 only.  The sample
    is sized from one calibration row so the whole --steps/--warmup run
    stays within ~3 minutes."""
    if rank != 0:
        return 0
    import numpy as np

    n = args.n or 16384
    rng = np.random.default_rng(0xB2000001)
    ys = rng.integers(-1000, 1001, (n, n)).astype(np.float64)
    ys[rng.random((n, n)) < 0.25] = math.inf
    cores = len(os.sched_getaffinity(0))
    btas = stock_reference()

    def make_x(rows):
        xs = rng.integers(-1000, 1001, (rows, n)).astype(np.float64)
        xs[rng.random((rows, n)) < 0.25] = math.inf
        return xs

    if btas is not None:
        MIN = btas.SemiringKind.MIN_PLUS
        Y = btas.TropicalMatrix(MIN, ys)
        tiles = btas.TileSpec(32, 32, cores)
        kind = "reference"

        def step(X):
            btas.matmul(X, Y, tiles=tiles)

        def prep(xs):
            return btas.TropicalMatrix(MIN, xs)

        what = f"btas.matmul(X, Y, tiles=TileSpec(32, 32, {cores})) (stock reference, byte-compiled oracle/_ref)"
    else:
        from oracle import tropical as ot

        yo = ot.orient(ot.MIN, ys)
        kind = "port"

        def step(X):
            ot.matmul(X, yo, ot.MIN, "f64", True, tile_rows=32, tile_cols=32, workers=cores)

        def prep(xs):
            return ot.orient(ot.MIN, xs)

        what = f"NumPy restatement of btas.matmul (thread pool of {cores})"
    # calibrate on one 32-row tile (the reference's throughput collapses on
    # thinner blocks: per-tile overhead), then take 64 rows if the whole
    # --steps/--warmup run still fits ~150 s
    x32 = prep(make_x(32))
    t = time.perf_counter()
    step(x32)
    t32 = time.perf_counter() - t
    total = max(1, args.steps + args.warmup)
    rows = 64 if 2 * t32 * total <= 150.0 else 32
    X = prep(make_x(rows))
    times = []
    for i in range(args.warmup + args.steps):
        t = time.perf_counter()
        step(X)
        if i >= args.warmup:
            times.append(time.perf_counter() - t)
    if not times:
        t = time.perf_counter()
        step(X)
        times.append(time.perf_counter() - t)
    pairs = rows * n * n
    value = pairs / statistics.median(times) / 1e9
    res = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(statistics.median(times) * 1e3, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": f"minplus_gemm_n{n}_i32", "n": n,
                   "sample": f"{rows} rows x {n} x {n} per step", "operands": "uniform integers in [-1000,1000]",
                   "infinity_fraction": 0.25},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"{rows} rows x {n} x {n} per step: {what}"},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(res), flush=True)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
