#!/usr/bin/env python
"""HRKAN PINN loss+grad step benchmark (BASELINE.json metric: collocation points/s per PINN
loss+grad step, fp32, and % of the FP32/tensor peak).

A step = one pass of the whole hot path over the synthetic collocation set of the workload:
hrkan_pinn_loss_grad (forward jet, residual, loss, reverse pass) + the data-parallel allreduce of
the flat [dL/dtheta | loss parts | flag] buffer (N > 1) + hrkan_adam_step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]

N > 1: under torchrun (WORLD_SIZE set) one process per GPU over NCCL; `--gpus N` without WORLD_SIZE builds
the library once and re-executes itself under torch.distributed.run with N local ranks.  Points are
sharded in contiguous blocks (strong scaling: the global set of the config is fixed, every rank gets 1/N
of it); parameters are checked bit-identical on every rank after init and after the timed steps.
Rank 0 prints ONE JSON line.  See DESIGN.md "Measurement" for every field.  `--dry-run` rehearses the
launcher and the DP step on CPU (gloo, stub net).
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import hrkan_inputs as HI  # noqa: E402

METRIC = "collocation points/s per PINN loss+grad step (fp32)"
UNIT = "points/s"
DEFAULT_CONFIG = "C5"


def peaks():
    """Roofline denominators: MEASURED_PEAKS.json (driver-written) else the profiling guide fallback."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"bf16": d.get("bf16_tflops", 1619.2), "bf16_sustained": d.get("bf16_tflops_sustained", 1350.0),
                "hbm": d.get("hbm_gbs", 6545.6), "sm_max_mhz": d.get("sm_max_mhz", 1965.0), "source": "measured"}
    return {"bf16": 1590.0, "bf16_sustained": 1400.0, "hbm": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback"}


# ------------------------------------------------------------------------------------------
# Algorithmic FLOPs per kernel class (the dense KAN matrix product over all B
# bases; the first layer is structured: 2*O*D*B + (C-1)*2*O*B per point).
# ------------------------------------------------------------------------------------------
def class_flops(w: HI.Workload, n_int: int, n_bi: int, c_int: int):
    B = w.B
    L = len(w.widths) - 1
    out = {}
    for l in range(L):
        I, O = w.widths[l], w.widths[l + 1]
        kind = "first" if l == 0 else ("last" if l == L - 1 else "hidden")
        for cls in ("fwd", "wgrad", "dgrad"):
            if cls == "dgrad" and l == 0:
                continue
            tot = 0
            for n, C in ((n_int, c_int), (n_bi, 1)):
                if l == 0:
                    per = 2 * O * w.D * B + (C - 1) * 2 * O * B
                else:
                    per = 2 * C * O * I * B
                tot += n * per
            key = f"{cls}_{kind}"
            out[key] = out.get(key, 0) + tot
    out["fused_step"] = sum(out.values())      # the one-launch tiny-net kernel does every layer
    return out


def tensor_core_layers(w: HI.Workload, engine: int) -> bool:
    """True when the hidden layers run on the tcgen05 kernels (libhrkan's tc_layer_ok rule)."""
    if w.pde in ("kawahara", "aniso"):          # generic jet engine: band-limited FFMA on every layer
        return False
    hidden = [(w.widths[l], w.widths[l + 1]) for l in range(1, len(w.widths) - 2)]
    return engine != 1 and bool(hidden) and all(O in (64, 128, 256) and I % 8 == 0 and
                                                (engine == 2 or I * w.B >= 256) and w.B >= 8 for I, O in hidden)


def interior_channels(w: HI.Workload) -> int:
    """Jet channels of the interior pass: Burgers (u, u_x, u_t, u_xx), Poisson 1 + 2D, Kawahara the Taylor-5
    jet (7), anisotropic the full Hessian jet 1 + D + D(D+1)/2."""
    if w.pde == "burgers":
        return 4
    if w.pde == "kawahara":
        return 7
    if w.pde == "aniso":
        return 1 + w.D + w.D * (w.D + 1) // 2
    return 1 + 2 * w.D


def pde_of(w: HI.Workload):
    from paper_2409_14248_b200 import pde_struct
    if w.pde == "kawahara":
        return pde_struct("kawahara", w.alpha, adv=w.adv, disp3=w.disp3, disp5=w.disp5)
    if w.pde == "aniso":
        return pde_struct("aniso", w.alpha, aniso=list(w.aniso))
    return pde_struct(w.pde, w.alpha, w.adv, w.visc)


# ------------------------------------------------------------------------------------------
# ------------------------------------------------------------------------------------------
# clocks during the timed region (nvidia-smi sampler)
# ------------------------------------------------------------------------------------------
_NVML_POLLER = r"""
import sys, threading, time, pynvml
pynvml.nvmlInit()
try:
    h = pynvml.nvmlDeviceGetHandleByPciBusId(sys.argv[1])
except Exception:
    h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[2]))
mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
stop, out = threading.Event(), []
def poll():
    while not stop.is_set():
        out.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                    pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(float(sys.argv[3]))
t = threading.Thread(target=poll); t.start()
print("ready", flush=True)
sys.stdin.read()                      # runs until the parent closes stdin
stop.set(); t.join()
bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
        "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
        "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
        "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
for sm, r in out:
    print(sm, mx, *[n for n, b in bits.items() if r & b])
"""


class ClockSampler:
    """Samples the SM clock and the throttle reasons while the timed region runs.  NVML is polled every
    millisecond by a separate process that buffers its samples until the region ends (so it neither
    competes for this interpreter's GIL nor misses the sub-10 ms C1/C2 regions); fallback nvidia-smi."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.sm, self.mx, self.reasons = [], None, set()
        self.source = "none"

    def _bus_id(self):
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.gpu)
            return f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        except Exception:
            return "none"

    def __enter__(self):
        if os.environ.get("BENCH_CLOCK_PERIOD_S") == "off":
            return self
        try:
            self.proc = subprocess.Popen([sys.executable, "-c", _NVML_POLLER, self._bus_id(), str(self.gpu),
                                          os.environ.get("BENCH_CLOCK_PERIOD_S", "0.001")],
                                         stdin=subprocess.PIPE, stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            if self.proc.stdout.readline().strip() == "ready":
                self.source = "nvml"
                return self
            self.proc.kill()
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.source = "nvidia-smi"
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if not self.proc:
            return
        if self.source == "nvml":
            try:
                text, _ = self.proc.communicate(input="", timeout=30)
            except Exception:
                self.proc.kill()
                return
            for line in text.splitlines():
                parts = line.split()
                if len(parts) >= 2:
                    self.sm.append(float(parts[0]))
                    self.mx = float(parts[1])
                    self.reasons.update(parts[2:])
            return
        self.proc.terminate()
        try:
            text, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            return
        for line in text.splitlines():
            parts = [p.strip() for p in line.strip().split(",")]
            if len(parts) < 7:
                continue
            try:
                self.sm.append(float(parts[0]))
                self.mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(self.NAMES, parts[3:7]):
                if v.lower().startswith("active"):
                    self.reasons.add(n)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.mx, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": self.source}



# ------------------------------------------------------------------------------------------
# CPU oracle (cpu_baseline and --impl reference): the float64 oracle as it stands, sharded over
# point blocks across a process pool on every host core (same arithmetic, global normalisers)
# ------------------------------------------------------------------------------------------
def host_cores() -> int:
    return len(os.sched_getaffinity(0))


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def oracle_sample(w: HI.Workload, ps: HI.PointSet, n_int: int):
    """A strided sample of the workload with ~n_int interior points and a proportional share of
    boundary/initial points (at least 1 each)."""
    s_int = max(1, len(ps.interior) // max(1, n_int))
    frac = (len(ps.interior) // s_int) / len(ps.interior)
    nb = max(1, int(round(ps.n_bi * frac)))
    s_bi = max(1, ps.n_bi // nb)
    return ps.subset(s_int, s_bi)


def _oracle_job(wkey: str, m: int, interior, bi, gbi, n_int_global: int, n_bi_global: int):
    """One shard of the oracle loss+grad (runs in a pool worker or in-process)."""
    from oracle import hrkan_oracle as O
    w = HI.WORKLOADS[wkey].with_m(m) if m != HI.WORKLOADS[wkey].m else HI.WORKLOADS[wkey]
    params = HI.random_params(w.widths, w.G, w.k, seed=HI.PARAM_SEED)
    if w.pde in ("kawahara", "aniso"):            # higher-order / mixed jets: the torch float64 oracle
        from oracle import hrkan_oracle_jets as OJ
        net = OJ.Net(w.widths, w.G, w.k, w.m, w.lo, w.hi)
        pde = ({"kind": "kawahara", "alpha": w.alpha, "adv": w.adv, "disp3": w.disp3, "disp5": w.disp5}
               if w.pde == "kawahara" else {"kind": "aniso", "alpha": w.alpha, "K": list(w.aniso)})
        f = HI.aniso_forcing(interior, w) if w.pde == "aniso" else None
        lp, lb, g = OJ.loss_grad(net, [(a.astype(np.float64), b.astype(np.float64)) for a, b in params], pde,
                                 interior, bi, gbi, n_int_global=n_int_global, n_bi_global=n_bi_global, forcing=f)
        return lp + lb
    net = O.Net(w.widths, w.G, w.k, w.m, w.lo, w.hi)
    pde = {"kind": w.pde, "alpha": w.alpha, "adv": w.adv, "visc": w.visc}
    lp, lb, g = O.loss_grad(net, params, pde, interior, bi, gbi, n_int_global=n_int_global, n_bi_global=n_bi_global)
    return lp + lb


def _pool_init():
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


class OracleRunner:
    """Times the oracle on a sample: single-threaded in-process, or split into `cores` contiguous point
    blocks evaluated concurrently by a spawn-context process pool (one BLAS thread per worker; the
    oracle's einsums are single-threaded C loops, so processes are how it uses the cores)."""

    def __init__(self, w: HI.Workload, cores: int):
        self.w, self.cores = w, max(1, cores)
        self.pool = None

    def __enter__(self):
        if self.cores > 1:
            from concurrent.futures import ProcessPoolExecutor
            import multiprocessing as mp
            saved = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}
            for k in saved:
                os.environ[k] = "1"
            try:
                self.pool = ProcessPoolExecutor(self.cores, mp_context=mp.get_context("spawn"), initializer=_pool_init)
                list(self.pool.map(int, range(4 * self.cores)))            # start every worker
                tiny = oracle_sample(self.w, HI.make_points(self.w), 8)
                self.run(tiny, parallel=True)                                # warm the imports
            finally:
                for k, v in saved.items():
                    if v is None:
                        os.environ.pop(k, None)
                    else:
                        os.environ[k] = v
        return self

    def __exit__(self, *a):
        if self.pool:
            self.pool.shutdown(cancel_futures=True)

    @staticmethod
    def _bi(sample):
        bi = sample.boundary if sample.initial is None else np.concatenate([sample.boundary, sample.initial])
        gbi = sample.g_boundary if sample.initial is None else np.concatenate([sample.g_boundary, sample.g_initial])
        return bi, gbi

    def run(self, sample, parallel: bool):
        """(seconds, points) of one oracle loss+grad over the sample."""
        bi, gbi = self._bi(sample)
        ni, nb = len(sample.interior), len(bi)
        t0 = time.perf_counter()
        if parallel and self.pool:
            from paper_2409_14248_b200.parallel import shard_range
            futs = []
            for r in range(self.cores):
                a, b = shard_range(ni, r, self.cores)
                c, d = shard_range(nb, r, self.cores)
                futs.append(self.pool.submit(_oracle_job, self.w.key.split("_")[0], self.w.m, sample.interior[a:b],
                                             bi[c:d], gbi[c:d], ni, nb))
            for f in futs:
                f.result()
        else:
            _oracle_job(self.w.key.split("_")[0], self.w.m, sample.interior, bi, gbi, ni, nb)
        return time.perf_counter() - t0, ni + nb

    def size_sample(self, ps, target_s: float):
        """Interior-point count whose single-threaded oracle run takes ~target_s (geometric probe)."""
        n = 8
        dt, _ = self.run(oracle_sample(self.w, ps, n), parallel=False)
        while dt < target_s / 8 and n < len(ps.interior):
            n = min(len(ps.interior), n * 4)
            dt, _ = self.run(oracle_sample(self.w, ps, n), parallel=False)
        return max(1, min(len(ps.interior), int(n * target_s / max(dt, 1e-4))))


def cpu_baseline(w: HI.Workload, ps: HI.PointSet, target_s: float):
    """SURVEY §8(d) protocol: every host core (process pool over point blocks) plus a 1-thread figure,
    with the CPU model.  ~target_s of single-thread work, then the same per-core work on all cores."""
    cores = host_cores()
    with OracleRunner(w, cores) as R:
        n1 = R.size_sample(ps, target_s / 3)
        s1 = oracle_sample(w, ps, n1)
        dt1, np1 = R.run(s1, parallel=False)
        sN = oracle_sample(w, ps, n1 * cores)
        dtN, npN = R.run(sN, parallel=True)
    desc = (f"{w.key} strided samples of the same synthetic set: {len(sN.interior)} interior + {sN.n_bi} "
            f"boundary/initial points split into {cores} contiguous blocks over a {cores}-process pool "
            f"(1-thread figure: {len(s1.interior)} + {s1.n_bi} points in-process); float64 numpy oracle loss+grad")
    return {"value": npN / dtN, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc, "seconds": dtN,
            "single_thread_value": np1 / dt1, "single_thread_seconds": dt1, "cpu_model": cpu_model()}


# ------------------------------------------------------------------------------------------
def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3, help=">= 3: step 0 loads modules")
    ap.add_argument("--config", default=os.environ.get("HRKAN_BENCH_CONFIG", DEFAULT_CONFIG))
    ap.add_argument("--m", type=int, default=None, help="override the HR order (C4 sweep)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--engine", type=int, default=0, help="0 auto, 1 SIMT only, 2 tensor cores")
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--graph", type=int, default=-1,
                    help="CUDA-graph replay of the loss+grad call: 1 on, 0 off, -1 auto (on for the launch-bound C1/C2)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--prof-steps", type=int, default=3, help="profiled steps (per-launch events) after the timed region")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU/gloo rehearsal of the N-rank launcher and the DP step with a stub net (no GPU)")
    return ap.parse_args(argv)


def workload(args) -> HI.Workload:
    w = HI.WORKLOADS[args.config]
    if args.m is not None:
        w = w.with_m(args.m)
    return w


def config_dict(w: HI.Workload, world: int, args, graph: bool) -> dict:
    return {"workload": w.key, "name": w.name, "n_interior": w.n_int, "n_boundary_initial": w.n_bnd + w.n_ic,
            "widths": list(w.widths), "G": w.G, "k": w.k, "m": w.m, "pde": w.pde, "parallelism": f"dp{world}",
            "l2": "flushed between timed steps (256 MiB write)", "engine": args.engine, "cuda_graph": graph}


def run_reference(args):
    """The reference arm for this tier = the float64 oracle as it stands, on the host cores (process pool
    over point blocks), each step a bounded strided sample of the same workload (rank 0 only; the other
    ranks exit without work)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    w = workload(args)
    ps = HI.make_points(w)
    cores = host_cores()
    per_step = max(1.0, 150.0 / max(1, args.steps + args.warmup))
    with OracleRunner(w, cores) as R:
        n1 = R.size_sample(ps, per_step / 2)
        sample = oracle_sample(w, ps, n1 * cores)
        times = []
        for s in range(args.warmup + args.steps):
            dt, npts = R.run(sample, parallel=True)
            if s >= args.warmup:
                times.append(dt)
    value = npts * len(times) / sum(times)
    desc = (f"{w.key} strided sample: {len(sample.interior)} interior + {sample.n_bi} boundary/initial points of the "
            f"same synthetic set, split into {cores} contiguous blocks over a {cores}-process pool; float64 numpy "
            f"oracle loss+grad per step")
    graph = (w.key in ("C1", "C2")) if args.graph < 0 else bool(args.graph)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict(w, args.gpus, args, graph),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc,
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# N-rank launcher: `bench.py --gpus N` with no WORLD_SIZE in the environment builds the library ONCE,
# then re-executes itself under torch.distributed.run with N local ranks (127.0.0.1 rendezvous).
# ------------------------------------------------------------------------------------------
def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def ensure_built(dry_run: bool) -> int:
    """Build libhrkan.so (sm_100a) if stale; returns 1 (a build check ran here).  The dry run only
    records the call (the CPU rehearsal must not depend on nvcc)."""
    if dry_run:
        print("[bench] build (dry run: not compiling)", file=sys.stderr, flush=True)
        return 1
    import __graft_entry__
    __graft_entry__.build(load=False)
    return 1


def launch_ranks(args, argv) -> int:
    n_built = ensure_built(args.dry_run)
    env = dict(os.environ, HRKAN_BENCH_BUILT=str(n_built), MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + list(argv)
    return subprocess.call(cmd, env=env, cwd=ROOT)


# ------------------------------------------------------------------------------------------
# dry-run stub: a CPU net with the HRKANNet call surface (host logic only, no HRKAN arithmetic)
# ------------------------------------------------------------------------------------------
class StubNet:
    """Linear least squares in place of the HRKAN loss: grad = 2/N_int sum_p (theta . phi(x_p)) phi(x_p)
    with phi = [1, x, x^2] per coordinate, + the boundary term; Adam replicated (torch CPU).  Exercises
    exactly what DPTrainStep does with a real net: shard-local evaluation with global normalisers, one
    allreduce, replicated optimiser, replica digests."""

    def __init__(self, D: int, seed: int):
        import torch
        g = torch.Generator().manual_seed(seed)
        self.n_params = 1 + 2 * D
        self.theta = torch.randn(self.n_params, generator=g, dtype=torch.float32)
        self.m = torch.zeros_like(self.theta)
        self.v = torch.zeros_like(self.theta)
        self.t = 0

    @staticmethod
    def _phi(x):
        import torch
        return torch.cat([torch.ones(len(x), 1, dtype=x.dtype), x, x * x], 1)

    def pinn_loss_grad(self, pde, interior, boundary, g_boundary, initial=None, g_initial=None, forcing=None,
                       n_int_global=None, n_bi_global=None, out=None):
        import torch
        out.zero_()
        for pts, tgt, n, k in ((interior, None, n_int_global, 0), (boundary, g_boundary, n_bi_global, 1),
                               (initial, g_initial, n_bi_global, 1)):
            if pts is None or len(pts) == 0:
                continue
            ph = self._phi(pts)
            r = ph @ self.theta - (0 if tgt is None else tgt)
            out[:self.n_params] += 2.0 / n * (ph.T @ r)
            out[self.n_params + k] += float((r * r).sum()) / n
        return out

    def adam_step(self, grad, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
        self.t += 1
        self.m.mul_(b1).add_((1 - b1) * grad)
        self.v.mul_(b2).add_((1 - b2) * grad * grad)
        self.theta -= lr * (self.m / (1 - b1 ** self.t)) / ((self.v / (1 - b2 ** self.t)).sqrt() + eps)

    def get_params(self):
        return self.theta.clone()


def run_rank(args):
    import torch
    import torch.distributed as dist
    from paper_2409_14248_b200.parallel import DPTrainStep, check_replicas, global_counts

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dry = args.dry_run
    if not dry:
        torch.cuda.set_device(local)
    if world > 1:
        if dry:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    # build once: by the launcher (HRKAN_BENCH_BUILT) or by local rank 0 while the others wait
    builds_here = 0
    if not os.environ.get("HRKAN_BENCH_BUILT"):
        if local == 0:
            builds_here = ensure_built(dry)
        if world > 1:
            dist.barrier()
    w = workload(args)
    ps = HI.make_points(w)
    sh = ps.shard(rank, world)
    n_int_g, n_bi_g = global_counts({"interior": ps.interior, "boundary": ps.boundary, "initial": ps.initial})
    if dry:
        dev = torch.device("cpu")
        net = StubNet(w.D, seed=HI.PARAM_SEED)
        pde = None
        graph = False
        stream = None
    else:
        import __graft_entry__  # noqa: F401  (the library is built; load it)
        from paper_2409_14248_b200 import HRKANNet, load_library
        load_library()
        dev = torch.device(f"cuda:{local}")
        net = HRKANNet(w.widths, w.G, w.k, w.m, w.lo, w.hi, seed=HI.PARAM_SEED, device=local)
        net.set_engine(args.engine)
        if args.chunk:
            net.set_chunk_points(args.chunk)
        pde = pde_of(w)
        graph = (w.key in ("C1", "C2")) if args.graph < 0 else bool(args.graph)
        # graph replay needs a non-legacy stream; eager runs use the current stream
        stream = torch.cuda.Stream(device=dev) if graph else torch.cuda.current_stream()
        torch.cuda.set_stream(stream)
        net.set_graph_mode(graph)
    same0, _ = check_replicas(net, world)
    cu = lambda a: None if a is None else torch.from_numpy(a).to(dev)
    dsets = {"interior": cu(sh.interior), "boundary": cu(sh.boundary), "g_boundary": cu(sh.g_boundary),
             "initial": cu(sh.initial), "g_initial": cu(sh.g_initial), "forcing": cu(sh.forcing)}
    npar = net.n_params
    out = torch.empty(npar + 4, dtype=torch.float32, device=dev)
    step = DPTrainStep(net, pde, dsets, n_int_g, n_bi_g, out, world=world)

    def sync():
        if not dry:
            torch.cuda.synchronize()

    def timer():
        """(start, stop, elapsed_ms) on the launching stream (CUDA events) or the host clock (dry run)."""
        if dry:
            box = {}
            return (lambda: box.__setitem__("a", time.perf_counter()),
                    lambda: box.__setitem__("b", time.perf_counter()),
                    lambda: 1000.0 * (box["b"] - box["a"]))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        return (lambda: a.record(stream), lambda: b.record(stream), lambda: a.elapsed_time(b))

    for s in range(args.warmup):
        step()
    sync()
    flush = None if dry else torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2

    def timed_region(n_steps, sets=None, result=None):
        evs = [timer() for _ in range(n_steps)]
        if world > 1:
            dist.barrier()
        sync()
        for s in range(n_steps):
            if flush is not None:
                flush.fill_(float(s))        # L2 flush between timed steps (outside the event pair)
            evs[s][0]()
            step(sets, result)
            evs[s][1]()
        sync()
        if world > 1:
            dist.barrier()
        ms = sum(e[2]() for e in evs) / n_steps
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)       # max over ranks
        return float(t.item())

    # ---------------- headline: device-resident inputs, no per-launch instrumentation
    launches0 = 0 if dry else net.launch_count()
    with ClockSampler(local) if not dry else _NullCtx() as clk:
        ms_max = timed_region(args.steps)
    launches = 0 if dry else net.launch_count() - launches0
    n_points = n_int_g + n_bi_g
    value = n_points / (ms_max / 1000.0)
    loss = float(out[npar:npar + 2].sum().item())
    flag = float(out[npar + 2].item())
    same1, digests = check_replicas(net, world)

    # ---------------- end to end: HOST (pinned) inputs through the C ABI, result read back
    e2e = None
    if not args.no_e2e:
        pin = (lambda a: None if a is None else torch.from_numpy(a)) if dry else \
              (lambda a: None if a is None else torch.from_numpy(a).pin_memory())
        hsets = {"interior": pin(sh.interior), "boundary": pin(sh.boundary), "g_boundary": pin(sh.g_boundary),
                 "initial": pin(sh.initial), "g_initial": pin(sh.g_initial), "forcing": pin(sh.forcing)}
        res = torch.empty(4, dtype=torch.float32)
        res = res if dry else res.pin_memory()
        h2d = sum(x.numel() * 4 for x in hsets.values() if x is not None)
        step(hsets, res)
        sync()
        ems = timed_region(args.steps, hsets, res)
        e2e = {"value": n_points / (ems / 1000.0), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": 16, "ms_per_step": ems}

    # ---------------- roofline: a second timed region of profiled steps (per-launch CUDA events on the
    # launching stream, eager), so the headline above carries no instrumentation
    roofline = None
    if not dry:
        roofline = measure_roofline(args, w, sh, net, step, stream, graph, ms_max)

    # ---------------- replica / build bookkeeping across ranks
    builds = [builds_here]
    if world > 1:
        builds = [None] * world
        dist.all_gather_object(builds, builds_here)
    total_builds = sum(builds) + int(os.environ.get("HRKAN_BENCH_BUILT", "0") or 0)

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1 and not dry:
            cpu = cpu_baseline(w, ps, args.cpu_seconds)
        comm = {"backend": "gloo" if dry else ("nccl" if world > 1 else None), "world_size": world}
        if world > 1 and not dry:
            comm["nccl_version"] = ".".join(map(str, torch.cuda.nccl.version()))
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
                # fp32 FFMA kernels; the wide-layer contractions run bf16x3 (bf16 hi/lo operands, fp32 TMEM accumulate)
                "vs_baseline": None, "dtype": "f32+bf16x3" if tensor_core_layers(w, args.engine) else "f32",
                "data": "synthetic" if not dry else "synthetic (dry run: CPU stub net, gloo)",
                "config": config_dict(w, world, args, graph),
                "e2e": e2e, "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu,
                "clocks": clk.summary() if not dry else None, "loss": loss, "nonfinite_flag": flag,
                "comm": comm, "replicas": {"params_identical_after_init": same0, "params_identical_after_steps": same1,
                                           "digest": digests[0][:16]},
                "builds": {"total": total_builds, "per_rank": builds},
                "step": "pinn_loss_grad + allreduce(N>1) + adam_step"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


class _NullCtx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def measure_roofline(args, w, sh, net, step, stream, graph, ms_headline):
    """Per-class device times from `--prof-steps` eager steps with per-launch CUDA events on the library
    stream; achieved = the dominant class's algorithmic FLOPs / its device time."""
    import torch
    n_prof = max(1, args.prof_steps)
    if graph:
        net.set_graph_mode(False)     # per-launch events need eager launches
    net.profile_enable(True)
    net.profile_read()
    for _ in range(n_prof):
        step()
    torch.cuda.synchronize()
    prof = net.profile_read()
    net.profile_enable(False)
    if graph:
        net.set_graph_mode(True)
    dominant = max(prof, key=lambda k: prof[k][0])
    pk = peaks()
    fl = class_flops(w, len(sh.interior), sh.n_bi, interior_channels(w))
    dom_ms, dom_n = prof[dominant]
    dom_flops = fl.get(dominant, 0) * n_prof
    clock_mhz = pk["sm_max_mhz"]
    n_sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    fp32_peak = n_sms * 128 * 2 * clock_mhz * 1e6 / 1e12     # SIMT (FFMA) peak
    achieved = dom_flops / (dom_ms / 1000.0) / 1e12 if dom_ms > 0 else 0.0
    if dominant in ("fwd_hidden", "wgrad_hidden", "dgrad_hidden") and tensor_core_layers(w, args.engine):
        peak, bound = pk["bf16_sustained"], "tensor"          # bf16x3 tcgen05 kernels: measured BF16 tensor peak
    else:
        peak, bound = fp32_peak, "alu"
    traffic, traffic_note = None, None
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", f"r02_ncu_{w.key.lower()}.json")))
        hit = [v for v in tj["kernels"].values() if v.get("class") == dominant]
        if hit and dom_n:
            pts_per_launch = (len(sh.interior) + sh.n_bi) * n_prof / dom_n
            traffic = max(hit, key=lambda v: v["time_ms"])["dram_bytes_per_point"] * pts_per_launch
            traffic_note = f"ncu dram bytes/point (profiles/r02_ncu_{w.key.lower()}.json) x points per launch"
    except (OSError, ValueError, KeyError):
        pass
    per_class = {k: v[0] / n_prof for k, v in prof.items() if v[1]}
    prof_step_ms = sum(per_class.values())
    return {"kernel_class": dominant, "bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak if peak else None, "traffic": traffic, "traffic_note": traffic_note,
            "launches": dom_n, "avg_launch_ms": dom_ms / max(1, dom_n),
            "share_of_step": (dom_ms / n_prof) / ms_headline if ms_headline > 0 else None,
            "algorithmic_flops_per_step": fl.get(dominant, 0),
            "peak_note": (f"FP32 FFMA = {n_sms} SMs x 128 lanes x 2 x {clock_mhz:.0f} MHz (derived)" if bound == "alu"
                          else f"BF16 dense sustained {pk['bf16_sustained']} TFLOP/s ({pk['source']} peak); "
                               f"achieved counts fp32-equivalent algorithmic FLOPs, bf16x3 issues 3 MMAs per "
                               f"product, so frac <= 1/3"),
            "per_class_ms_per_step": per_class, "profiled_kernel_ms_per_step": prof_step_ms,
            "events": f"{n_prof} eager steps after the timed region, per-launch CUDA events on the library stream"}


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    if args.impl == "reference":
        run_reference(args)
        return 0
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return launch_ranks(args, argv)
    run_rank(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
