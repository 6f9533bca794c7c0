"""Benchmark: 1080p SSIM & MS-SSIM frame-pairs/s on B200 (BASELINE.json metric, config 2 workload).

One step = one pass of the hot path over one batch of 64 synthetic 1080p u8
frame pairs (config 2: seeded 1/f noise vs 8x8-DCT quantisation, step
U[4, 40]): per frame the Gaussian 11/1.5 SSIM (score, l_mean, cs_mean) and
the 5-scale MS-SSIM (standard exponents, product), scale 0 shared.

  value   : frames resident in HBM (device-timed with CUDA events, max over ranks)
  e2e     : same work through the public host API (HostBatchScorer): pinned
            host frames -> H2D (inside the timed region) -> kernels -> D2H scores
  roofline: the dominant kernel (level-0 fused Gaussian SSIM) against the FP32
            FFMA peak measured in-run (MEASURED_PEAKS.json carries no FP32 entry)
  cpu_baseline: the numpy oracle port (same algorithms as the reference) on all
            host cores, bounded sample

Multi-GPU (torchrun): weak scaling, each rank scores its own 64 frames; no
collective on the data path; ranks meet only at the barriers around the timed
region and in one all_reduce(MAX) of the elapsed time.

--gpus N without torchrun: bench.py re-launches itself under
torch.distributed.run with N ranks (one per GPU, 127.0.0.1 rendezvous); each
rank binds its host threads to its GPU's NUMA node before it pins its frames.

--impl reference: times the reference's own CPU implementation (ssimkit,
installed untracked under baseline/_ref by tools/install_reference.sh; the
oracle port when that is absent) on the host cores for the same metric and
config; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "1080p SSIM & MS-SSIM frame-pairs/sec at 1/2/4/8 B200; % of roofline"
UNIT = "frame-pairs/s"
BATCH = 64
H, W = 1080, 1920
K, SIGMA, LEVELS = 11, 1.5, 5
WORKLOAD = "config2: 64x 1920x1080 u8 pairs (1/f noise vs 8x8 DCT quantisation), Gaussian 11/1.5 SSIM + 5-scale MS-SSIM per pair, scale 0 shared"


def frame_indices(rank: int) -> range:
    return range(rank * BATCH, (rank + 1) * BATCH)


def _gen(i: int):
    from paper_2101_06354_b200 import synth

    return synth.dct_pair(2, i, H, W)


def generate(indices, workers: int):
    import numpy as np
    from concurrent.futures import ProcessPoolExecutor

    if workers <= 1:
        pairs = [_gen(i) for i in indices]
    else:
        with ProcessPoolExecutor(workers) as ex:
            pairs = list(ex.map(_gen, indices, chunksize=2))
    ref = np.stack([p[0] for p in pairs])
    dist = np.stack([p[1] for p in pairs])
    return ref, dist


# ---------------------------------------------------------------------------
# CPU baseline (oracle port; test infrastructure used only as the measured baseline)
# ---------------------------------------------------------------------------

REF_DIR = REPO / "baseline" / "_ref"


def _reference_impl():
    """The reference package itself (pure Python ssimkit under baseline/_ref) when it is
    installed, else the oracle port of its numpy algorithms.  Returns (kind, score_fn)."""
    if (REF_DIR / "ssimkit" / "__init__.py").exists():
        if str(REF_DIR) not in sys.path:
            sys.path.insert(0, str(REF_DIR))
        import ssimkit
        from ssimkit.config import MultiscaleSpec, SsimConfig, WindowSpec

        cfg = SsimConfig(window=WindowSpec.gaussian(SIGMA, k=K))
        spec = MultiscaleSpec.product(LEVELS)

        def score(a, b):
            ssimkit.ssim_score(a, b, cfg)       # the reference's public API, stock code path
            ssimkit.msssim(a, b, cfg, spec)
            return 1.0

        return "reference", score
    from oracle import ssim_oracle as O

    win = dict(shape="gauss", k=K, sigma=SIGMA)

    def score(a, b):
        O.ssim_terms(a, b, **win)       # ssim_score path (the reference computes it separately)
        O.msssim(a, b, LEVELS, **win)   # msssim path
        return 1.0

    return "port", score


_SCORE = None


def _cpu_score(pair) -> float:
    """One frame pair through the reference's CPU path: ssim_score + msssim (Gaussian 11/1.5)."""
    global _SCORE
    if _SCORE is None:
        _SCORE = _reference_impl()[1]
    return _SCORE(*pair)


def _cpu_warm(_) -> int:
    global _SCORE
    _SCORE = _reference_impl()[1]  # imports outside the timed region
    return os.getpid()


def cpu_kind() -> str:
    return "reference" if (REF_DIR / "ssimkit" / "__init__.py").exists() else "port"


class CpuBaseline:
    """A persistent pool of single-threaded worker processes running the reference's CPU path.

    Inputs are generated up front and worker start-up/imports happen before any timing, so the
    timed region holds only the reference algorithm (plus pickling the 4 MB pair to a worker).
    """

    def __init__(self, workers: int):
        from concurrent.futures import ProcessPoolExecutor

        single_threaded_blas()
        self.workers = workers
        self.pool = ProcessPoolExecutor(workers)
        list(self.pool.map(_cpu_warm, range(workers)))

    def rate(self, pairs) -> tuple[float, float]:
        t0 = time.perf_counter()
        done = sum(self.pool.map(_cpu_score, pairs))
        wall = time.perf_counter() - t0
        return done / wall, wall

    def close(self):
        self.pool.shutdown()


def single_threaded_blas() -> None:
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"


def cpu_context(pairs, cores: int) -> dict:
    """The two context figures SURVEY.md 8(d) asks for beside the all-process rate: one core
    (one pair in this process) and the reference's own frame-parallel mechanism, a
    ThreadPoolExecutor over the frames (src/pipeline.py:319-322), with `cores` threads."""
    from concurrent.futures import ThreadPoolExecutor

    _cpu_warm(0)
    t0 = time.perf_counter()
    _cpu_score(pairs[0])
    one = time.perf_counter() - t0
    t0 = time.perf_counter()
    with ThreadPoolExecutor(cores) as ex:
        done = sum(ex.map(_cpu_score, pairs))
    tp = time.perf_counter() - t0
    return {"single_core": {"value": 1.0 / one, "unit": UNIT, "cores": 1, "sample": "1 config-2 pair"},
            "thread_pool": {"value": done / tp, "unit": UNIT, "cores": cores,
                            "sample": f"{len(pairs)} config-2 pairs on a {cores}-thread ThreadPoolExecutor "
                                      "(the reference's frame-parallel mechanism, src/pipeline.py:319-322)"}}


def cpu_pairs(n: int, workers: int):
    ref, dist = generate(range(10_000, 10_000 + n), workers)
    return [(ref[i], dist[i]) for i in range(n)]


def host_cores() -> int:
    """Usable host cores: the affinity mask, capped by a cgroup CPU quota if one is set."""
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count() or 1
    try:
        quota, period = Path("/sys/fs/cgroup/cpu.max").read_text().split()[:2]
        if quota != "max":
            n = min(n, max(1, int(float(quota) / float(period))))
    except (OSError, ValueError):
        pass
    return n


def host_info() -> dict:
    model = None
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "usable_cores": host_cores()}


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0:  # sampling live before timing starts
                time.sleep(0.02)
        except OSError:
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

    def summary(self) -> dict:
        import statistics

        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# flop count
# ---------------------------------------------------------------------------

def ssim_flops(h: int, w: int, k: int = K, s: int = 1) -> float:
    ho, wo = (h - k) // s + 1, (w - k) // s + 1
    return 3.0 * h * w + h * wo * 5 * k * 2 + ho * wo * 5 * k * 2 + ho * wo * 22


def msssim_flops(h: int, w: int, levels: int = LEVELS) -> float:
    total, hh, ww = 0.0, h, w
    for lv in range(levels):
        if lv:
            hh, ww = hh // 2, ww // 2
            total += 8.0 * hh * ww
        total += ssim_flops(hh, ww)
    return total


# ---------------------------------------------------------------------------

def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def bench_config(world: int) -> dict:
    """The workload dict, identical in both arms (the driver compares them)."""
    return {"workload": WORKLOAD, "batch": BATCH, "h": H, "w": W, "window": "gauss 11/1.5",
            "levels": LEVELS, "seed_base": 202, "parallelism": f"frame-shard x{world} (weak)",
            "l2": "inputs 265 MB per step > 126 MB L2 (no flush needed)"}


def _free_port() -> int:
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def relaunch_if_needed(args) -> None:
    """`bench.py --gpus N` outside torchrun: re-exec under torch.distributed.run with N ranks
    (one process per GPU).  Under torchrun the world size must equal --gpus."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        return
    if args.gpus <= 1 or args.impl == "reference":
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def gpu_numa_cpus(device_index: int):
    """(numa node, cpu list) of the GPU's PCI device from sysfs, or (None, None)."""
    import torch

    p = torch.cuda.get_device_properties(device_index)
    bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    try:
        node = int(Path(f"/sys/bus/pci/devices/{bus}/numa_node").read_text())
    except (OSError, ValueError):
        return None, None
    if node < 0:
        return None, None
    try:
        spec = Path(f"/sys/devices/system/node/node{node}/cpulist").read_text().strip()
    except OSError:
        return node, None
    cpus = set()
    for part in spec.split(","):
        lo, _, hi = part.partition("-")
        cpus.update(range(int(lo), int(hi or lo) + 1))
    return node, sorted(cpus)


def bind_numa(device_index: int) -> dict:
    """Bind this rank's host threads (and so the first touch of its pinned frames) to the
    CPUs of its GPU's NUMA node."""
    node, cpus = gpu_numa_cpus(device_index)
    if not cpus:
        return {"numa_node": node, "bound": False}
    try:
        allowed = os.sched_getaffinity(0)
        use = [c for c in cpus if c in allowed]
        if use:
            os.sched_setaffinity(0, use)
            return {"numa_node": node, "bound": True, "cpus": len(use)}
    except (AttributeError, OSError):
        pass
    return {"numa_node": node, "bound": False}


def launch_selftest(args) -> None:
    """CPU check of the launcher: every rank joins a gloo group and rank 0 prints who came up."""
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    dist.init_process_group("gloo")
    t = torch.tensor([rank, local, os.getpid()], dtype=torch.int64)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    if rank == 0:
        print(json.dumps({"n_gpus": world, "ranks": [int(x[0]) for x in out],
                          "local_ranks": [int(x[1]) for x in out],
                          "pids": len({int(x[2]) for x in out})}), flush=True)
    dist.destroy_process_group()


def run_reference(args) -> None:
    world, rank, _ = dist_env()
    if rank != 0:
        return
    single_threaded_blas()
    cores = host_cores()
    per_step = cores  # one pair per worker process per step
    pairs = cpu_pairs(per_step, cores)
    cpu = CpuBaseline(cores)
    # warm-up steps run the same algorithm on 256x512 crops of the step's pairs (worker
    # imports, allocator and caches warmed; a full 1080p step is several s of CPU per pair)
    crops = [(a[:256, :512].copy(), b[:256, :512].copy()) for a, b in pairs]
    for _ in range(args.warmup):
        cpu.rate(crops)
    t_total = 0.0
    for _ in range(args.steps):
        _, wall = cpu.rate(pairs)
        t_total += wall
    cpu.close()
    value = per_step * args.steps / t_total
    kind = cpu_kind()
    what = ("the reference package itself (ssimkit from baseline/_ref: ssim_score + msssim per pair)"
            if kind == "reference" else "oracle port of ssimkit's numpy path (ssim_score + msssim per pair)")
    cpu_base = {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                "sample": f"{per_step} config-2 pairs per step (1 per single-threaded worker process), {what}",
                "host": host_info()}
    if not args.no_cpu_context:
        cpu_base.update(cpu_context(pairs, cores))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": max(world, args.gpus),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": bench_config(max(world, args.gpus)),
        "sample_pairs_per_step": per_step,
        "cpu_baseline": cpu_base,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200(args) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2101_06354_b200 as P
    from paper_2101_06354_b200 import _native, engine

    world, rank, local = dist_env()
    if world > torch.cuda.device_count():
        sys.exit(f"bench.py: {world} ranks but only {torch.cuda.device_count()} visible GPU(s)")
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", torch.cuda.current_device())
    numa = bind_numa(dev.index)  # before any host buffer is allocated or pinned
    lib = _native.load_library()
    cores = host_cores()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    gen_workers = max(1, cores // max(1, world))
    ref_np, dist_np = generate(frame_indices(rank), gen_workers)
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(SIGMA, k=K))
    spec = P.MultiscaleSpec.product(LEVELS)
    ref_dev = torch.from_numpy(ref_np).to(dev)
    dist_dev = torch.from_numpy(dist_np).to(dev)

    def step():
        return P.msssim_batch(ref_dev, dist_dev, cfg, spec, with_ssim=True)

    clk = ClockSampler(dev.index).__enter__()  # sampled across every timed region below
    # ---- device-resident throughput (value) ----
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    l0 = int(lib.ssk_launch_count())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        out = step()
    e1.record()
    torch.cuda.synchronize()
    launches = int(lib.ssk_launch_count()) - l0
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    ms_per_step = ms / args.steps
    value = world * BATCH * args.steps / (ms / 1e3)
    ms_score, ss_terms = out
    scores_host = ms_score.cpu().numpy()
    assert np.all(np.isfinite(scores_host))

    # ---- dominant kernel: level-0 fused Gaussian SSIM over the batch ----
    pair = engine.device_pair(ref_dev, dist_dev, 8, gauss=True)
    want = _native.WANT_Q | _native.WANT_L | _native.WANT_CS
    for _ in range(3):
        engine.ssim(pair, cfg.window, cfg.c1, cfg.c2, want)
    reps = 20
    torch.cuda.synchronize()
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record()
    for _ in range(reps):
        engine.ssim(pair, cfg.window, cfg.c1, cfg.c2, want)
    k1.record()
    torch.cuda.synchronize()
    # each engine.ssim = 1 fused kernel + 1 tiny fold kernel; the fold is < 1% (see profiles/)
    kernel_ms = k0.elapsed_time(k1) / reps
    flops = BATCH * ssim_flops(H, W)
    achieved = flops / (kernel_ms * 1e-3) / 1e12
    peak = ctypes_probe(lib, 2.0)
    roofline = {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": committed_traffic(), "kernel": "gauss_levels_kernel<11, u8, 4, classic, 256> (level-0 score launch over the 64-frame batch, wide strips, 2 CTAs/SM; the MS-SSIM step runs the same kernel with the fused level-1 stores)",
                "kernel_ms": kernel_ms, "flops_per_launch": flops,
                "peak_source": "measured in-run: FFMA probe (ssk_probe_fp32_tflops, 2 s sustained); "
                               "MEASURED_PEAKS.json has no FP32 entry",
                "step_flops": BATCH * msssim_flops(H, W),
                "step_frac": BATCH * msssim_flops(H, W) / (ms_per_step * 1e-3) / 1e12 / peak}

    # ---- end to end through the host API (pinned host frames, H2D + D2H inside the timed region) ----
    ref_host = torch.from_numpy(ref_np).pin_memory()
    dist_host = torch.from_numpy(dist_np).pin_memory()
    scorer = P.batch.HostBatchScorer(cfg, spec, mode="both", chunk=8)
    for _ in range(max(1, args.warmup)):
        scorer(ref_host, dist_host)
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    pending = None
    for _ in range(args.steps):  # each step submitted one ahead of reading the previous step's scores
        nxt = scorer.submit(ref_host, dist_host)
        if pending is not None:
            ms_h, ss_h = pending.result()
        pending = nxt
    ms_h, ss_h = pending.result()
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    e2e = {"value": world * BATCH * args.steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": scorer.h2d_bytes,
           "d2h_bytes_per_step": scorer.d2h_bytes, "ms_per_step": 1e3 * e2e_s / args.steps,
           "path": "HostBatchScorer.submit per step, one step ahead (pinned host -> chunked async H2D on a copy stream -> msssim_batch(with_ssim) -> D2H into pinned host -> result())"}
    clk.__exit__(None, None, None)
    assert np.array_equal(ms_h, scores_host), "host-API and device-batch scores differ"

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        n_cpu = cores * args.cpu_pairs_per_core
        pool = CpuBaseline(cores)
        sample = cpu_pairs(n_cpu, cores)
        rate, wall = pool.rate(sample)
        pool.close()
        kind = cpu_kind()
        what = "ssimkit itself from baseline/_ref" if kind == "reference" else "oracle port of ssimkit's numpy path"
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": kind,
               "sample": f"{n_cpu} config-2 pairs ({args.cpu_pairs_per_core} per single-threaded process), "
                         f"ssim_score + msssim each, {what}, {wall:.1f} s wall", "host": host_info()}
        if not args.no_cpu_context:
            cpu.update(cpu_context(sample[:cores], cores))

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
            "config": bench_config(world), "host_binding": numa,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "check": {"msssim_mean": float(scores_host.mean()),
                                                "ssim_mean": float(ss_terms.score.mean().item())},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def ctypes_probe(lib, seconds: float) -> float:
    import ctypes

    import torch

    out = ctypes.c_double(0.0)
    rc = lib.ssk_probe_fp32_tflops(seconds, ctypes.byref(out), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    if rc != 0:
        raise RuntimeError(f"fp32 probe failed: {rc}")
    return out.value


def committed_traffic():
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture, if any."""
    p = REPO / "profiles" / "roofline_traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            return None
    return None


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-pairs-per-core", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cpu-context", action="store_true", help="skip the 1-core / thread-pool CPU figures")
    ap.add_argument("--launch-selftest", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    relaunch_if_needed(args)
    if args.launch_selftest:
        launch_selftest(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
