"""Benchmark: one ACI Hadamard product of BASELINE.json configs[3] at chi = 256 per step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--chi 256] [--impl ours|reference]

A step is one full aci_elementwise call (canonicalisation + 4 iterations of L->R / R->L 2-site
updates + output cores) over device-resident inputs. `value` is the contraction-model FP64
TFLOP/s aggregated over ranks; `ms_per_step` is the wall time of one product
(device time, CUDA events on the call's stream). L2 is flushed (256 MiB write) between timed
steps, outside the timed region. Multi-GPU runs independent replicas (one
product does not shard), `scaling` = "weak".

--impl reference times the CPU oracle (oracle/, naive-loop C, single thread) on a bounded
sample of the same workload (the first iterations), rank 0 only.
"""
import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ACI Hadamard-product wall time (ms) and FP64 TFLOP/s vs χ; fraction of FP64 peak"
UNIT = "TFLOP/s (FP64, contraction model)"


def _file_peaks():
    """HBM copy bandwidth from the driver-written MEASURED_PEAKS.json (it has no FP64 entry)."""
    try:
        m = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return {"hbm_gbs": m.get("hbm_gbs"), "hbm_source": "MEASURED_PEAKS.json"}
    except Exception:
        return {"hbm_gbs": 6650.0, "hbm_source": "fallback (B200_PROFILING.md)"}


def measure_prrlu_latency(sizes=(64, 128, 256, 512, 1024)):
    """Per-pivot latency of the library's prrLU on seeded square blocks of each tier (m x m, up to
    512 pivots), with the work and without it (ACI_PRRLU_NOWORK: the exchange chain alone — CTA
    argmax, cluster key exchange, cross-cluster leg, column read — the design's per-pivot floor),
    measured in this run through libaci_peak.so (csrc/peak_probe.cu; best of 3 launches)."""
    import ctypes
    from paper_2604_00037_b200 import _build
    lib = ctypes.CDLL(_build.build_peak())
    lib.aci_peak_prrlu.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                   ctypes.POINTER(ctypes.c_int)]
    out = {}
    for m in sizes:
        row = {}
        for key, nowork in (("kernel_us", 0), ("floor_us", 1)):
            v, piv = ctypes.c_double(0.0), ctypes.c_int(0)
            rc = lib.aci_peak_prrlu(m, nowork, 3, ctypes.byref(v), ctypes.byref(piv))
            row[key] = v.value if rc == 0 else None
            row["pivots"] = piv.value
        out[m] = row
    return out


def measure_prrlu_latency_shapes(log, dims, maxrank):
    """Per-pivot time of the library's prrLU with and without the rank-1 update + rescan
    (ACI_PRRLU_NOWORK) on seeded blocks of EVERY (live m x n, pivots r) shape of one product's pivot
    log, each launched for its bond's static size as the product launches it (so tier choice and
    the hand-off are those of the product); returns (floor_ms, kernel_ms, per-shape rows), both
    weighted by the log's pivot counts."""
    import ctypes
    from paper_2604_00037_b200 import _build
    lib = ctypes.CDLL(_build.build_peak())
    lib.aci_peak_prrlu_shape.argtypes = [ctypes.c_int] * 6 + [ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                                                ctypes.POINTER(ctypes.c_int)]
    L = len(dims)

    def rmax(b):  # csrc/aci.cu: min(maxrank, prod d[0..b], prod d[b+1..L-1])
        lo = hi = 1
        for t in range(b + 1):
            lo = min(lo * dims[t], 1 << 30)
        for t in range(b + 1, L):
            hi = min(hi * dims[t], 1 << 30)
        return min(maxrank, lo, hi)

    shapes = {}
    for e in log:
        b = e["bond"]
        m, n = dims[b] * e["rl"], dims[b + 1] * e["rr"]
        sm = dims[b] * (1 if b == 0 else rmax(b - 1))
        sn = dims[b + 1] * (1 if b == L - 2 else rmax(b + 1))
        key = (m, n, max(e["r"], 1), sm, sn)
        shapes[key] = shapes.get(key, 0) + e["r"]
    rows, floor_ms, kern_ms = [], 0.0, 0.0
    for (m, n, r, sm, sn), cnt in sorted(shapes.items(), key=lambda kv: -kv[1]):
        row = {"m": m, "n": n, "r": r, "static": [sm, sn], "pivots": cnt}
        for key, nowork in (("kernel_us", 0), ("floor_us", 1)):
            v, piv = ctypes.c_double(0.0), ctypes.c_int(0)
            rc = lib.aci_peak_prrlu_shape(m, n, r, sm, sn, nowork, 3, ctypes.byref(v), ctypes.byref(piv))
            row[key] = v.value if rc == 0 else None
        if row["floor_us"]:
            floor_ms += cnt * row["floor_us"] / 1e3
        if row["kernel_us"]:
            kern_ms += cnt * row["kernel_us"] / 1e3
        rows.append(row)
    return floor_ms, kern_ms, rows


def _block_tier(m, n):
    """The probe size whose tier a live m x n block runs in (prrlu.cu variant lists)."""
    big = max(m, n)
    for t in (64, 128, 256, 512):
        if big <= t:
            return t
    return 1024


def measure_peaks(stream=None):
    """FP64 roofline denominators measured IN THIS RUN on this GPU (MEASURED_PEAKS.json has no FP64
    entry): cuBLAS DGEMM 8192^3 through torch.matmul (best of 5 after a warm-up, CUDA events), the
    DMMA register loop and the DFMA register loop of libaci_peak.so (paper_2604_00037_b200/csrc/
    peak_probe.cu; best of 5 launches over all SMs)."""
    import ctypes
    import torch
    from paper_2604_00037_b200 import _build
    p = _file_peaks()
    lib = ctypes.CDLL(_build.build_peak())
    lib.aci_peak_fp64.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    for kind, key in ((0, "dmma_tflops"), (1, "dfma_tflops")):
        v = ctypes.c_double(0.0)
        rc = lib.aci_peak_fp64(kind, 5, ctypes.byref(v))
        p[key] = v.value if rc == 0 else None
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.matmul(a, b)
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 2.0 * n ** 3 / (e0.elapsed_time(e1) * 1e9))
    del a, b, c
    torch.cuda.empty_cache()
    p["dgemm_tflops"] = best
    p["source"] = ("measured in this bench run: cuBLAS DGEMM 8192^3 (torch.matmul float64), DMMA / DFMA "
                   "register loops over all SMs (csrc/peak_probe.cu); best of 5")
    return p


class ClockSampler:
    """nvidia-smi clocks sampled every 100 ms on a reader thread; start() returns once the first
    sample has arrived, so even a short timed region is covered."""

    def __init__(self, gpu_index=0):
        self.proc = None
        self.gpu = gpu_index
        self.lines = []
        self.thread = None

    def start(self):
        import threading
        import time
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return

        def read():
            for line in self.proc.stdout:
                self.lines.append((time.monotonic(), line))

        self.thread = threading.Thread(target=read, daemon=True)
        self.thread.start()
        t0 = time.monotonic()
        while not self.lines and time.monotonic() - t0 < 5.0 and self.proc.poll() is None:
            time.sleep(0.01)
        self.t_begin = time.monotonic()

    def stop(self):
        import time
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t_end = time.monotonic()
        time.sleep(0.12)  # the sample covering the end of the timed region
        self.proc.terminate()
        if self.thread is not None:
            self.thread.join(timeout=2.0)
        # samples taken during the timed region (the one just before it stands in if it was shorter)
        inside = [ln for t, ln in self.lines if self.t_begin - 0.1 <= t <= t_end + 0.11]
        out = inside or [ln for _, ln in self.lines[-1:]]
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


def run_reference(args):
    """The oracle (CPU, single thread) as the reference arm: every TIMED step is the whole
    workload (configs[3] at --chi, all 4 iterations: the same config as our arm); the untimed
    warm-up steps run iteration 1 only (a CPU program has no warm-up effect worth a 27 s product),
    so --steps K --warmup W costs about K whole products."""
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    import oracle
    from workloads import make_config
    cf = make_config(3, args.chi, npts=0)
    times, flops = [], []
    for i in range(args.warmup + args.steps):
        sweeps = cf["max_sweeps"] if i >= args.warmup else 1
        t0 = time.perf_counter()
        res = oracle.aci(cf["inputs"], cf["op"], cf["y_init"], cf["tol"], cf["maxrank"], sweeps)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
            flops.append(res.report["flops_contraction"])
        res.free()
    tot_t, tot_f = sum(times), sum(flops)
    value = tot_f / tot_t / 1e12
    sample = (f"configs[3] chi={args.chi}: the whole product (all {cf['max_sweeps']} iterations) per timed step, "
              f"naive-loop C oracle on 1 thread of {os.cpu_count()} host cores ({_cpu_model()}); "
              f"contraction-model flops / wall time")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference", "same_config": True,
            "config": {"workload": cf["name"], "chi": args.chi, "L": 40, "d": 2, "maxrank": cf["maxrank"],
                       "tol": cf["tol"], "iterations": cf["max_sweeps"], "parallelism": "replicas",
                       "l2": "n/a (CPU)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "host_cores": os.cpu_count(),
                             "cpu_model": _cpu_model(), "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _ncu_traffic():
    """DRAM bytes per launch (read + write) of the dominant kernels, from the newest committed
    `ncu --set full` capture summary under profiles/ (None if there is none)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_summary.json")))
    if not files:
        return {}
    out = {}
    for f in reversed(files):  # newest capture of each kernel class
        d = json.load(open(f))
        for k, v in d.items():
            if (isinstance(v, dict) and "dram_bytes_read" in v and "dram_bytes_write" in v
                    and (k.startswith("prrlu_r") or k.startswith("gemmpi"))):
                key = "prrlu" if k.startswith("prrlu") else "contraction"
                if key not in out:
                    out[key] = {"bytes": v["dram_bytes_read"] + v["dram_bytes_write"], "source": os.path.basename(f),
                                "kernel": v["kernel"]}
    return out


def reduce_over_ranks(ms, flops, e2e_value, dist, device):
    """Replica aggregation: the job time is the slowest rank's, the work is summed."""
    if dist is None:
        return ms, flops, e2e_value
    import torch
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    f = torch.tensor([flops, e2e_value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(f, op=dist.ReduceOp.SUM)
    return float(t.item()), float(f[0].item()), float(f[1].item())


def cpu_baseline(chi, sweeps):
    import oracle
    from workloads import make_config
    cf = make_config(3, chi, npts=0)
    t0 = time.perf_counter()
    res = oracle.aci(cf["inputs"], cf["op"], cf["y_init"], cf["tol"], cf["maxrank"], sweeps)
    dt = time.perf_counter() - t0
    v = res.report["flops_contraction"] / dt / 1e12
    res.free()
    return {"value": v, "unit": UNIT, "cores": 1, "host_cores": os.cpu_count(), "cpu_model": _cpu_model(),
            "kind": "oracle",
            "sample": f"configs[3] chi={chi}, {sweeps} of 4 iterations (4 = the whole product), single-thread naive C oracle, "
                      f"{dt:.1f} s on 1 of {os.cpu_count()} host cores ({_cpu_model()})"}


def _free_port():
    import socket
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    return port


def launch_ranks(n, argv):
    """`bench.py --gpus N` outside torchrun: re-launch this script as N ranks (one process per GPU)
    under torch.distributed.run on 127.0.0.1; the ranks assert WORLD_SIZE == N. NCCL's
    communicator log stays on (NCCL_DEBUG=INFO unless set)."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + argv
    return subprocess.call(cmd, env=env)


def run_dry(args):
    """--dry-run: the multi-rank plumbing on CPU (gloo), for tests: every rank times the CPU oracle
    on configs[0] as its 'product', the line aggregates over ranks exactly as the GPU path does
    (max time, summed work) and reports n_gpus = the ranks that ran."""
    import torch.distributed as tdist
    ws, rank, _ = _dist()
    dist = None
    if ws > 1:
        tdist.init_process_group("gloo")
        dist = tdist
    import oracle
    from workloads import make_config
    cf = make_config(0, npts=0)
    tot, fl = 0.0, 0.0
    for i in range(args.warmup + args.steps):
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        r = oracle.aci(cf["inputs"], cf["op"], cf["y_init"], cf["tol"], cf["maxrank"], cf["max_sweeps"])
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            tot += 1e3 * dt
            fl += r.report["flops_contraction"]
        r.free()
    t_max, f_sum, _ = reduce_over_ranks(tot, fl, 0.0, dist, "cpu")
    world = dist.get_world_size() if dist is not None else 1
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": f_sum / t_max / 1e9, "unit": UNIT, "n_gpus": world,
                          "ranks_ran": world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": t_max / args.steps, "dry_run": True, "scaling": "weak",
                          "config": {"workload": cf["name"], "parallelism": f"replicas x{world}"}}), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--chi", type=int, default=256)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-sweeps", type=int, default=4, help="cpu_baseline sample: oracle iterations (4 = whole)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="CPU/gloo multi-rank plumbing check (tests)")
    ap.add_argument("--no-chi-sweep", action="store_true", help="skip the chi = 64, 128 products")
    ap.add_argument("--no-complex", action="store_true", help="skip the complex Fourier-series sweep")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    ws, rank, local = _dist()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        if not args.dry_run:
            import torch
            if torch.cuda.device_count() < args.gpus:
                print(json.dumps({"error": f"--gpus {args.gpus} but {torch.cuda.device_count()} visible GPUs"}))
                return 2
        return launch_ranks(args.gpus, sys.argv[1:])
    if "WORLD_SIZE" in os.environ and args.impl == "ours" and ws != args.gpus:
        print(json.dumps({"error": f"WORLD_SIZE={ws} but --gpus {args.gpus}"}), flush=True)
        return 2
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import paper_2604_00037_b200 as aci
    from workloads import make_config

    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    aci.load()
    # a dedicated (non-default) stream: the library captures each iteration as a CUDA graph
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream

    def run_chi(chi, steps, warmup, with_e2e):
        cf = make_config(3, chi, npts=0)
        xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
        y0 = aci.TensorTrain.from_cores(cf["y_init"])
        flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
        for _ in range(warmup):
            out, st, rep, _ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"],
                                                  y_init=y0, stream=sptr)
            out.free()
        torch.cuda.synchronize()
        sampler = ClockSampler(local)
        sampler.start()
        tot_ms, tot_flops, launches = 0.0, 0.0, 0
        prof_tot = {}
        reps = []
        for i in range(steps):
            flush.fill_(float(i))
            torch.cuda.synchronize()
            if dist is not None:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            out, st, rep, ex = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"],
                                                   y_init=y0, stream=sptr)
            e1.record(stream)
            torch.cuda.synchronize()
            tot_ms += e0.elapsed_time(e1)
            tot_flops += rep["flops_contraction"]
            launches += rep["n_launches"]
            reps.append(rep)
            out.free()
        clocks = sampler.stop()
        # per-kernel-class device times: the same product once more with CUDA events around every
        # launch on the call's stream (direct launches instead of the graph; not part of `value`)
        for i in range(max(1, steps // 2)):
            flush.fill_(float(i))
            torch.cuda.synchronize()
            out, st, rep, ex = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"],
                                                   y_init=y0, stream=sptr, profile=True)
            torch.cuda.synchronize()
            for k, v in ex["profile"].items():
                p = prof_tot.setdefault(k, {"ms": 0.0, "launches": 0, "runs": 0})
                p["ms"] += v["ms"]
                p["launches"] += v["launches"]
                p["runs"] += 1
            prof_rep = rep
            out.free()
        for p in prof_tot.values():
            p["ms"] /= p["runs"]
            p["launches"] //= p["runs"]
        e2e = None
        if with_e2e:
            e2e = run_e2e(cf, steps, sptr)
            # sanity gate on the timed workload: the product against f of the inputs on 10^4 seeded
            # multi-indices (R16); the parity tests compare with the oracle itself
            smp = make_config(3, chi, npts=10_000)["samples"]
            out, st, rep, _ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"],
                                                  y_init=y0, stream=sptr)
            ref = np.prod([x.evaluate(smp) for x in xs], axis=0)
            err = float(np.abs(out.evaluate(smp) - ref).max() / np.abs(ref).max())
            out.free()
            e2e["rel_max_err_vs_f_of_inputs"] = err
            e2e["within_10_tol"] = bool(err <= 10 * cf["tol"])
        return cf, tot_ms, tot_flops, launches, prof_tot, reps, clocks, e2e

    def run_e2e(cf, steps, sptr):
        """Same product through the public C-ABI from pinned host buffers: H2D of the inputs and
        y_init (tt_create), the product, D2H of every output core (tt_get_cores)."""
        pinned_in = []
        for t in list(cf["inputs"]) + [cf["y_init"]]:
            pc = []
            for c in t.cores:
                buf = torch.empty(c.shape, dtype=torch.float64, pin_memory=True)
                buf.numpy()[...] = c
                pc.append(buf.numpy())
            pinned_in.append(pc)
        h2d = sum(c.nbytes for pc in pinned_in for c in pc)
        tot, d2h = 0.0, 0
        out_bufs = None
        for i in range(steps + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            hx = [aci.TensorTrain.from_cores(pc) for pc in pinned_in[:-1]]
            hy = aci.TensorTrain.from_cores(pinned_in[-1])
            out, st, rep, _ = aci.aci_elementwise(cf["op"], hx, cf["tol"], cf["maxrank"], cf["max_sweeps"],
                                                  y_init=hy, stream=sptr)
            d, r = out.shape()
            if out_bufs is None or [b.shape for b in out_bufs] != [(r[s], d[s], r[s + 1]) for s in range(len(d))]:
                out_bufs = [torch.empty((r[s], d[s], r[s + 1]), dtype=torch.float64, pin_memory=True).numpy()
                            for s in range(len(d))]
            import ctypes as C
            ptrs = (C.POINTER(C.c_double) * len(d))(*[b.ctypes.data_as(C.POINTER(C.c_double)) for b in out_bufs])
            aci._binding._check(aci.load().tt_get_cores(out.handle, ptrs))
            dt = time.perf_counter() - t0
            out.free()
            for h in hx + [hy]:
                h.free()
            if i > 0:  # first iteration is the e2e warm-up
                tot += dt
                d2h = sum(b.nbytes for b in out_bufs)
                fl = rep["flops_contraction"]
        return {"value": fl * steps / tot / 1e12, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * tot / steps}

    def run_complex(Ks, steps):
        """Complex values: the paper's random Fourier series product
        (configs[5] with K+1 coefficients) timed like the main workload; error against
        the closed-form product on 2000 seeded points."""
        pts = []
        for K in Ks:
            cf = make_config(5, K, npts=2000)
            xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
            y0 = aci.TensorTrain.from_cores(cf["y_init"])
            for _ in range(2):
                out, st, rep, _ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"],
                                                      y_init=y0, stream=sptr)
                out.free()
            torch.cuda.synchronize()
            tot = 0.0
            for _ in range(steps):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                out, st, rep, _ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"],
                                                      y_init=y0, stream=sptr)
                e1.record(stream)
                torch.cuda.synchronize()
                tot += e0.elapsed_time(e1)
            smp = cf["samples"]
            x = (smp * (2.0 ** -np.arange(1, smp.shape[1] + 1))).sum(axis=1)
            g = [np.exp(1j * np.outer(x, np.arange(len(t.meta["coefs"])))) @ t.meta["coefs"] for t in cf["inputs"]]
            exact = g[0] * g[1]
            err = float(np.abs(out.evaluate(smp) - exact).max() / np.abs(exact).max())
            ms = tot / steps
            pts.append({"K": K, "chi_in": max(cf["inputs"][0].ranks), "chi_out": rep["max_rank"], "ms_per_product": ms,
                        "tflops": rep["flops_contraction"] / ms / 1e9, "pivots": rep["pivot_steps"],
                        "iterations": rep["iterations"], "rel_err_vs_closed_form": err, "tol": cf["tol"]})
            out.free()
        return {"workload": "cfg5_fourier_complex_L30 (P:289-311), f = g1 g2, tol 1e-8, maxrank 256",
                "points": pts,
                "note": "complex parity workload (NEXT-1); flops counted as 4x the real contraction model "
                        "(complex products)"}

    def run_all_configs(reps=2):
        """Every BASELINE.json config (and the complex configs[5]) once more: device ms per product
        (CUDA events, after one warm-up), iterations, pivots, max rank, and the relative max error
        against f applied to the inputs' values on 10^4 seeded points (R16)."""
        rows = []
        for cfg, arg in ((0, 0), (1, 0), (2, 0), (3, 64), (4, 0), (5, 4000)):
            cf = make_config(cfg, arg, npts=10_000)
            xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
            handles, op = xs, cf["op"]
            if cfg == 2:  # psi^3 with three aliased handles, merged by the library
                handles, op = [xs[0]] * 3, {"coef": [1.0], "expo": [[1, 1, 1]]}
            y0 = aci.TensorTrain.from_cores(cf["y_init"])
            out, st, rep, _ = aci.aci_elementwise(op, handles, cf["tol"], cf["maxrank"], cf["max_sweeps"],
                                                  y_init=y0, stream=sptr)
            out.free()
            tot = 0.0
            for _ in range(reps):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                out, st, rep, _ = aci.aci_elementwise(op, handles, cf["tol"], cf["maxrank"], cf["max_sweeps"],
                                                      y_init=y0, stream=sptr)
                e1.record(stream)
                torch.cuda.synchronize()
                tot += e0.elapsed_time(e1)
            smp = cf["samples"]
            vals = [x.evaluate(smp) for x in xs]
            ref = sum(c * np.prod([vals[n] ** e for n, e in enumerate(ex_)], axis=0)
                      for c, ex_ in zip(cf["op"]["coef"], cf["op"]["expo"]))
            err = float(np.abs(out.evaluate(smp) - ref).max() / np.abs(ref).max())
            rows.append({"config": cf["name"], "ms_per_product": tot / reps, "iterations": rep["iterations"],
                         "converged": bool(rep["converged"]), "pivots": rep["pivot_steps"],
                         "max_rank": rep["max_rank"], "tol": cf["tol"], "rel_max_err_vs_f_of_inputs": err,
                         "within_10_tol": bool(err <= 10 * cf["tol"]) if cfg != 4 else None,
                         "tflops": rep["flops_contraction"] / (tot / reps) / 1e9})
            out.free()
        return rows

    def run_steady(chis, iters=6):
        """Steady-state full-rank iterations: configs[3] run for `iters`
        iterations so that the last one is at the saturated ranks (2 chi); its device time
        (CUDA events around the iteration's graph) and its contraction-model flops (from the
        update log) per half-sweep."""
        pts = []
        for chi in chis:
            cf = make_config(3, chi, npts=0)
            xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
            y0 = aci.TensorTrain.from_cores(cf["y_init"])
            best = None
            for _ in range(3):
                out, st, rep, ex = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], iters, y_init=y0,
                                                       stream=sptr, log=True, iter_times=True)
                out.free()
                last = ex["iter_ms"][-1]
                best = last if best is None else min(best, last)
            L, nb = 40, 39
            tail = ex["log"][-2 * nb:]
            fl = 0.0
            for e in tail:
                b, rl, rr = e["bond"], e["rl"], e["rr"]
                m, n = 2 * rl, 2 * rr
                for xr in ([1] + [chi] * (L - 1) + [1], [1] + [2] * (L - 1) + [1]):
                    c0, c1, c2 = xr[b], xr[b + 1], xr[b + 2]
                    fl += 2.0 * rl * c0 * 2 * c1 + 2.0 * c1 * 2 * c2 * rr + 2.0 * m * c1 * n
            pts.append({"chi": chi, "iteration": len(ex["iter_ms"]), "ms_per_half_sweep": best / 2,
                        "gflop_per_half_sweep": fl / 2 / 1e9, "tflops": fl / best / 1e9,
                        "pivots_per_half_sweep": sum(e["r"] for e in tail) / 2,
                        "max_rank": max(e["r"] for e in tail)})
        lx = np.log([p["chi"] for p in pts])
        fit = lambda ys: float(np.polyfit(lx, np.log(ys), 1)[0])
        return {"points": pts, "exponent_half_sweep_time": fit([p["ms_per_half_sweep"] for p in pts]),
                "exponent_half_sweep_flops": fit([p["gflop_per_half_sweep"] for p in pts]),
                "note": "last iteration of a run allowed 6 (it converges once the ranks saturate at 2 chi): "
                        "contraction work per half-sweep scales as chi^3; the wall time grows slower "
                        "because the prrLU (one exchange per pivot, pivots ~ chi) dominates"}

    def run_concurrent(chi=64, ks=(1, 2, 4, 8), reps=3):
        """Product-level concurrency: k independent configs[3] products, each
        on its own stream from its own host thread with aci_options.concurrent (single-cluster
        prrLU launches, safe to co-schedule); products per second vs k (wall clock around the
        batch, device work only: inputs resident)."""
        import threading
        cf = make_config(3, chi, npts=0)
        pts = []
        for k in ks:
            streams = [torch.cuda.Stream() for _ in range(k)]
            data = [([aci.TensorTrain.from_cores(t) for t in cf["inputs"]], aci.TensorTrain.from_cores(cf["y_init"]))
                    for _ in range(k)]

            def work(i, n):
                xs, y0 = data[i]
                for _ in range(n):
                    out, *_ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"],
                                                  y_init=y0, stream=streams[i].cuda_stream, concurrent=True)
                    out.free()

            ths = [threading.Thread(target=work, args=(i, 1)) for i in range(k)]  # warm-up (graphs)
            [t.start() for t in ths]
            [t.join() for t in ths]
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ths = [threading.Thread(target=work, args=(i, reps)) for i in range(k)]
            [t.start() for t in ths]
            [t.join() for t in ths]
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            pts.append({"streams": k, "products": k * reps, "seconds": dt, "products_per_s": k * reps / dt,
                        "ms_per_product_amortised": 1e3 * dt / (k * reps)})
        base = pts[0]["products_per_s"]
        for p in pts:
            p["speedup_vs_1"] = p["products_per_s"] / base
        return {"workload": cf["name"],
                "mode": "aci_options.concurrent (single-cluster prrLU; blocks beyond one cluster: the cooperative "
                        "L2 grid tier)", "points": pts}

    def run_rook(chis=(64, 128), reps=3):
        """Rook pivoting (reading R23) against full pivoting on configs[3]:
        device ms per product (CUDA events), pivots, us per pivot (prrLU class time / pivots, from a
        profiled run), the reported error estimate and the relative max error against the exact
        product on 10^4 seeded samples. Rook covers blocks up to 512 rows (chi <= 128)."""
        pts = []
        for chi in chis:
            cf = make_config(3, chi, npts=10_000)
            xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
            y0 = aci.TensorTrain.from_cores(cf["y_init"])
            s = cf["samples"]
            exact = np.prod([x.evaluate(s) for x in xs], axis=0)
            for piv in ("full", "rook"):
                out, st, rep, _ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"],
                                                      y_init=y0, stream=sptr, pivoting=piv)
                out.free()
                tot = 0.0
                for _ in range(reps):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    out, st, rep, _ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"],
                                                          y_init=y0, stream=sptr, pivoting=piv)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    tot += e0.elapsed_time(e1)
                    err = float(np.abs(out.evaluate(s) - exact).max() / np.abs(exact).max())
                    out.free()
                o2, _, r2, ex2 = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"],
                                                     y_init=y0, stream=sptr, pivoting=piv, profile=True)
                o2.free()
                pts.append({"chi": chi, "pivoting": piv, "ms_per_product": tot / reps, "pivots": rep["pivot_steps"],
                            "us_per_pivot": 1e3 * ex2["profile"]["prrlu"]["ms"] / max(r2["pivot_steps"], 1),
                            "iterations": rep["iterations"], "converged": bool(rep["converged"]),
                            "error_estimate": rep["error_estimate"], "rel_max_err_vs_exact": err,
                            "max_rank": rep["max_rank"]})
        return {"workload": "cfg3_randomTT_L40 (chi 64, 128), f = ab", "points": pts,
                "note": "full pivoting stays the default (P:529); rook changes the pivots (R23) and is limited to "
                        "blocks of one CTA or one 16-CTA cluster (<= 512 rows)"}

    # the metric is quoted vs chi (B:2, configs[3]): time the chi = 64 and 128 products as well
    sweep = []
    if not args.no_chi_sweep:
        for chi in (64, 128):
            cf_, ms, fl, _, prof_, reps_, _, _ = run_chi(chi, max(2, args.steps // 2), args.warmup, False)
            n_ = max(2, args.steps // 2)
            sweep.append({"chi": chi, "ms_per_product": ms / n_, "tflops": fl / ms / 1e9,
                          "pivots": reps_[-1]["pivot_steps"], "flops_contraction": reps_[-1]["flops_contraction"],
                          "prrlu_ms": prof_["prrlu"]["ms"], "contraction_ms": prof_["gemm_pi"]["ms"] +
                          prof_["gemm_ab"]["ms"]})

    cf, tot_ms, tot_flops, launches, prof, reps, clocks, e2e = run_chi(args.chi, args.steps, args.warmup,
                                                                       with_e2e=True)
    steady = run_steady((64, 128, 256)) if (ws == 1 and not args.no_chi_sweep) else None
    allcfg = run_all_configs() if (ws == 1 and not args.no_chi_sweep) else None
    conc = None
    if ws == 1 and not args.no_chi_sweep:
        conc = run_concurrent()
        conc = {"chi64": conc, "chi256": run_concurrent(chi=256, ks=(1, 2, 4), reps=2)}
        conc["chi256"]["default_tier_ms_per_product"] = tot_ms / args.steps
    rook = run_rook() if (ws == 1 and not args.no_chi_sweep) else None
    cplx = None
    if ws == 1 and not args.no_complex:
        cplx = run_complex((1000, 4000, 16000), max(2, args.steps // 2))
    # max over ranks for time, sum over ranks for work (independent replicas)
    t_max, f_sum, e2e_sum = reduce_over_ranks(tot_ms, tot_flops, e2e["value"] if e2e else 0.0, dist, "cuda")
    if e2e is not None:
        e2e["value"] = e2e_sum
    pk = measure_peaks()  # after the timed regions: the same process, clocks and GPU
    lat, piv_by_tier, lat_shapes = None, {}, None
    if rank == 0:
        lat = measure_prrlu_latency()
        cfl = make_config(3, args.chi, npts=0)
        xs_ = [aci.TensorTrain.from_cores(t) for t in cfl["inputs"]]
        y0_ = aci.TensorTrain.from_cores(cfl["y_init"])
        o_, _, _, ex_ = aci.aci_elementwise(cfl["op"], xs_, cfl["tol"], cfl["maxrank"], cfl["max_sweeps"], y_init=y0_,
                                            stream=sptr, log=True)
        o_.free()
        for e in ex_["log"]:
            t = _block_tier(2 * e["rl"], 2 * e["rr"])
            piv_by_tier[t] = piv_by_tier.get(t, 0) + e["r"]
        lat_shapes = measure_prrlu_latency_shapes(ex_["log"], cfl["inputs"][0].d, cfl["maxrank"])
    if rank == 0:
        value = f_sum / t_max / 1e9  # GFLOP/ms -> TFLOP/s
        steps = args.steps
        r0 = reps[-1]
        # dominant kernel class by summed event time
        dom = max(prof, key=lambda k: prof[k]["ms"])
        pr = prof["prrlu"]
        pi = prof["gemm_pi"]
        prrlu_flops = reps[-1]["flops_prrlu"]  # per product; prof_tot is per product too
        pi_flops = reps[-1]["flops_contraction"]  # a3 dominates; a1/a2 included
        # per-pivot latency against the measured exchange floor of each block size, weighted by the
        # product's own pivot distribution (pivot log of one product)
        lat_fr = None
        if lat is not None and piv_by_tier:
            floor_ms = sum(cnt * lat[t]["floor_us"] for t, cnt in piv_by_tier.items() if lat[t]["floor_us"]) / 1e3
            kern_ms = sum(cnt * lat[t]["kernel_us"] for t, cnt in piv_by_tier.items() if lat[t]["kernel_us"]) / 1e3
            lat_fr = {"floor_ms_per_product": floor_ms, "probe_kernel_ms_per_product": kern_ms,
                      "product_prrlu_ms": pr["ms"], "frac": floor_ms / pr["ms"] if pr["ms"] else None,
                      "pivots_by_block": {str(k): v for k, v in sorted(piv_by_tier.items())},
                      "by_block": {str(k): v for k, v in lat.items()}}
            if lat_shapes is not None:
                # the same floor per (m, n, r) shape of the product's own log, launched for each bond's
                # static size (tiers and hand-off as in the product): this one is reported as 'frac'
                sf, sk, srows = lat_shapes
                lat_fr = dict(lat_fr, **{
                    "floor_ms_per_product": sf, "probe_kernel_ms_per_product": sk,
                    "frac": sf / pr["ms"] if pr["ms"] else None,
                    "square_blocks": {"floor_ms_per_product": floor_ms, "probe_kernel_ms_per_product": kern_ms,
                                      "frac": floor_ms / pr["ms"] if pr["ms"] else None,
                                      "note": "seeded m x m blocks by max(m, n) class (round-2 method)"},
                    "by_shape_top": srows[:12]})
        roof_prrlu = {"kernel": "prrlu_kernel (a5)", "bound": "alu",
                      "achieved": prrlu_flops / (pr["ms"] * 1e9) if pr["ms"] else None,
                      "peak": pk["dfma_tflops"], "unit": "TFLOP/s",
                      "frac": (prrlu_flops / (pr["ms"] * 1e9)) / pk["dfma_tflops"] if pr["ms"] else None,
                      "traffic": None, "per_launch_us": 1e3 * pr["ms"] / max(pr["launches"], 1),
                      "per_pivot_us": 1e3 * pr["ms"] / max(reps[-1]["pivot_steps"], 1),
                      "latency": dict(lat_fr or {}, **{
                          "per_pivot_us": 1e3 * pr["ms"] / max(reps[-1]["pivot_steps"], 1),
                          "floor_source": "measured in this run: the library's prrLU with the rank-1 update and "
                                          "rescan compiled out (csrc/peak_probe.cu, ACI_PRRLU_NOWORK) on seeded "
                                          "blocks of every (m, n, r) shape of the product's pivot log, each in its "
                                          "bond's static launch (tiers and hand-off as in the product), i.e. the "
                                          "exchange chain alone per pivot; weighted by the log's pivots; frac = "
                                          "floor / product prrLU time"}),
                      "note": "latency-bound: one cluster/L2 exchange per pivot (DESIGN.md §5); 'frac' above is "
                              "against the DFMA register loop measured in this run (peaks.dfma_tflops), "
                              "'latency.frac' against the measured exchange floor"}
        roof_pi = {"kernel": "gemm_dmma_kernel<fused f> (a3+a4) + a1/a2", "bound": "tensor",
                   "achieved": pi_flops / ((pi["ms"] + prof["gemm_ab"]["ms"]) * 1e9),
                   "peak": pk["dmma_tflops"], "unit": "TFLOP/s",
                   "frac": pi_flops / ((pi["ms"] + prof["gemm_ab"]["ms"]) * 1e9) / pk["dmma_tflops"],
                   "traffic": None, "note": "FP64 DMMA (mma.sync m8n8k4); peak = the DMMA register loop measured "
                                            "in this run (peaks.dmma_tflops); peaks.dgemm_tflops = cuBLAS DGEMM "
                                            "8192^3 in this run. The time is the event-timed sum over the contraction "
                                            "launches of the profiled run: it includes the streamed-Pi kernel's whole "
                                            "residency beside the prrLU (it waits for pivot rows), so this is a lower "
                                            "bound on the GEMMs' own rate; the serialised ncu launch list "
                                            "(profiles/r02zl_chi256_launches_summary.txt) has ~10.5 ms of contraction "
                                            "kernels per chi = 256 product"}
        tr = _ncu_traffic()
        if "prrlu" in tr:
            roof_prrlu["traffic"] = tr["prrlu"]["bytes"]
            roof_prrlu["traffic_source"] = tr["prrlu"]["source"] + ": " + tr["prrlu"]["kernel"]
        if "contraction" in tr:
            roof_pi["traffic"] = tr["contraction"]["bytes"]
            roof_pi["traffic_source"] = tr["contraction"]["source"] + ": " + tr["contraction"]["kernel"]
        roof = roof_prrlu if dom == "prrlu" else roof_pi
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": steps,
            "warmup": args.warmup, "ms_per_step": t_max / steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cf["name"], "chi": args.chi, "L": 40, "d": 2, "maxrank": cf["maxrank"],
                       "tol": cf["tol"], "iterations": cf["max_sweeps"], "parallelism": f"replicas x{ws}",
                       "l2": "flushed (256 MiB write) between steps"},
            "roofline": roof,
            "roofline_kernels": {"prrlu": roof_prrlu, "contraction": roof_pi},
            "kernel_ms_per_step": {k: v["ms"] for k, v in prof.items()},
            "kernel_ms_note": "per-class CUDA-event sums from an extra profiled run of the same product "
                              "(events around every launch, no graph); value/ms_per_step come from the "
                              "unprofiled timed steps",
            "fraction_of_fp64_peak_end_to_end": value / ws / pk["dmma_tflops"],
            "clocks": clocks,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "product": {"iterations": r0["iterations"], "converged": bool(r0["converged"]),
                        "max_rank": r0["max_rank"], "pivot_steps": r0["pivot_steps"],
                        "flops_contraction": r0["flops_contraction"], "flops_prrlu": r0["flops_prrlu"],
                        "error_estimate": r0["error_estimate"]},
            "peaks": pk,
        }
        if sweep:
            pts = sweep + [{"chi": args.chi, "ms_per_product": t_max / steps / ws, "tflops": value / ws,
                            "pivots": r0["pivot_steps"], "flops_contraction": r0["flops_contraction"],
                            "prrlu_ms": prof["prrlu"]["ms"],
                            "contraction_ms": prof["gemm_pi"]["ms"] + prof["gemm_ab"]["ms"]}]
            lx = np.log([p["chi"] for p in pts])
            fit = lambda ys: float(np.polyfit(lx, np.log(ys), 1)[0])
            line["chi_sweep"] = {"points": pts,
                                 "exponent_wall_time": fit([p["ms_per_product"] for p in pts]),
                                 "exponent_contraction_flops": fit([p["flops_contraction"] for p in pts]),
                                 "exponent_contraction_kernel_time": fit([p["contraction_ms"] for p in pts]),
                                 "note": "fixed 4-iteration runs from a rank-2 y_init: the contraction work is "
                                         "sub-cubic here because ranks saturate late (SURVEY 8(d)); the pivot "
                                         "count grows ~linearly in chi"}
        if steady is not None:
            line["steady_state_half_sweep"] = steady
        if allcfg is not None:
            line["all_configs"] = allcfg
        if conc is not None:
            line["concurrent_products"] = conc
        if rook is not None:
            line["rook_pivoting"] = rook
        if cplx is not None:
            line["complex_fourier"] = cplx
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args.chi, args.ref_sweeps)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
