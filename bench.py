#!/usr/bin/env python3
"""Benchmark driver (replaces the reference's proj/benchmarks/bench.cpp).

Workload (BASELINE config 4): Jacobi-2D 5-point, fp64, 32768 x 32768 per GPU,
T = 512 steps, zero Dirichlet ring, F = init_value("F", flat) (reference
exec.cpp:21-28).  One "step" = one full T=512 run of the hot path.
  --gpus N (torchrun, one rank per GPU): rows are sharded; weak scaling keeps
  32768 rows per rank (global grid 32768N x 32768), halo rows exchanged with
  NCCL send/recv every bt steps, overlapped with the interior.

Metric: stencil GUpdates/s (whole job), plus
  roofline  — dominant kernel s2d5 (16 algorithmic bytes per cell per launch,
              i.e. 16/bt B/update) vs the measured HBM copy bandwidth;
  e2e       — the same metric through the C ABI with host buffers: every step
              copies F in from pinned host memory and Out back
              (pcotgpu_run_batch: the copies of adjacent steps overlap compute);
  cpu_baseline — the reference's own tiled CPU path (its emitted C, OpenMP,
              all host cores) on a bounded sample, rank 0, N=1.
  per_config — BASELINE configs 0-3 in the same run (N=1, rank 0): each
              through the executor's default schedule, CUDA-event timed with
              an L2 flush before every timed run, clocks sampled, output
              checksum against the reference golden (config 3: 4096 sampled
              cells of the reference's result, componentwise 1e-12), roofline
              fraction, and the reference's CPU path on a bounded sample.
--impl reference runs only that reference CPU path (rank 0) on the sample.
--gpus N without torchrun re-launches itself under torch.distributed.run with
N ranks (NCCL_DEBUG=INFO); --dry-run checks the rank plumbing on CPU (gloo).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

EMIT_DIR = os.path.join(REPO, "oracle", "_ref", "emit")
SAMPLE = "jacobi2d_N8192_T160"
SAMPLE_INIT = "jacobi2d_N8192_T0"
SAMPLE_UPDATES = 8192 * 8192 * 160
METRIC = "stencil GUpdates/s at 1/2/4/8 B200; % HBM roofline; DRAM bytes/update"  # BASELINE.json


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peak_hbm():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(bt, cells):
    """dram__bytes_read.sum + dram__bytes_write.sum per s2d5 launch, from the
    committed `ncu --set full` capture of this bench command at this depth
    (profiles/ncu_bench_s2d5_bt<bt>_r*.json; tools/ncu_summary.py)."""
    import glob

    for p in sorted(glob.glob(os.path.join(REPO, "profiles", "ncu_bench_s2d5_bt%d_r*.json" % bt)),
                    reverse=True):
        try:
            with open(p) as f:
                d = json.load(f)
            if abs(d.get("algorithmic_bytes", 0) - 16.0 * cells) < 1:
                return {"bytes_per_launch": d["dram_bytes"],
                        "over_algorithmic": d.get("traffic_over_algorithmic"),
                        "source": os.path.relpath(p, REPO)}
        except Exception:
            continue
    return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + q,
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        sms, mx, reasons = [], None, set()
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                sms.append(float(f[1]))
                mx = float(f[2])
                names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
                for n, v in zip(names, f[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
        except Exception:
            pass
        finally:
            try:
                os.unlink(self.path)
            except OSError:
                pass
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sms)}


def run_reference_sample(threads, sample=SAMPLE, init=SAMPLE_INIT, leaf=None):
    """Wall time of the reference's emitted C on a sample minus its init-only
    twin; `leaf` overrides the binary's default leaf sizes (argv b0..)."""
    env = dict(os.environ)
    env["OMP_NUM_THREADS"] = str(threads)

    def wall(tag, argv):
        b = os.path.join(EMIT_DIR, tag)
        t0 = time.perf_counter()
        out = subprocess.run([b] + argv, capture_output=True, text=True, env=env, check=True)
        return time.perf_counter() - t0, out.stdout.split()[1]

    t_init, _ = wall(init, [])
    t_run, chk = wall(sample, [str(x) for x in leaf] if leaf else [])
    return max(t_run - t_init, 1e-9), chk


# leaf sizes (t, rows, cols) tried for the OpenMP sample; the best is the baseline
LEAF_SWEEP = [(16, 128, 1024), (32, 128, 512), (8, 256, 2048)]
SEQ_SAMPLE, SEQ_INIT, SEQ_UPDATES = "jacobi2d_N4096_T32_seq", "jacobi2d_N4096_T0_seq", 4096 * 4096 * 32


def cpu_baseline_port(threads):
    """Fallback when oracle/_ref was not shipped: the oracle port on the sample."""
    from tests import oracle_ctypes as O

    O.lib().oracle_set_threads(threads)
    F = O.init_array("F", 8192 * 8192)
    t0 = time.perf_counter()
    O.stencil2d5(8192, 160, 0, F)
    return time.perf_counter() - t0


def reference_available():
    return os.path.exists(os.path.join(EMIT_DIR, SAMPLE)) and os.path.exists(
        os.path.join(EMIT_DIR, SAMPLE_INIT))


def host_info():
    info = {"nproc": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    info["cpu_model"] = line.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as f:
            info["mem_total_gib"] = round(int(f.readline().split()[1]) / 2**20, 1)
    except OSError:
        pass
    return info


def cpu_baseline(threads):
    """Best of a leaf sweep of the reference's OpenMP path on the sample, plus
    its sequential emitted C on a smaller sample (same rule)."""
    sweep, seq = [], None
    if reference_available():
        for leaf in LEAF_SWEEP:
            secs, chk = run_reference_sample(threads, leaf=leaf)
            sweep.append({"leaf": list(leaf), "seconds": round(secs, 3), "checksum": chk,
                          "GUpdates/s": round(SAMPLE_UPDATES / secs / 1e9, 4)})
        best = min(sweep, key=lambda e: e["seconds"])
        secs, chk, kind = best["seconds"], best["checksum"], "reference"
        if os.path.exists(os.path.join(EMIT_DIR, SEQ_SAMPLE)):
            ssecs, _ = run_reference_sample(1, SEQ_SAMPLE, SEQ_INIT)
            seq = {"value": SEQ_UPDATES / ssecs / 1e9, "unit": "GUpdates/s", "cores": 1,
                   "seconds": round(ssecs, 3),
                   "sample": "Jacobi-2D 4096^2, T=32, reference emitted C without OpenMP"}
    else:
        secs, chk = cpu_baseline_port(threads), None
        kind = "port"
    return {"value": SAMPLE_UPDATES / secs / 1e9, "unit": "GUpdates/s", "cores": threads,
            "kind": kind, "seconds": round(secs, 3), "checksum": chk,
            "sample": "Jacobi-2D 8192^2, T=160 (same rule/ring/init as config 4; "
                      "reference emitted recursive C, OpenMP tasks, -O2 -ffp-contract=off; "
                      "wall minus init-only run; best of the leaf sweep)",
            "leaf_sweep": sweep, "sequential": seq, "host": host_info()}


def reference_arm(args, rank, world):
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    times = []
    kind = "reference" if reference_available() else "port"
    # warm-up steps walk the leaf sweep; the timed steps use the fastest leaf
    warm = {}
    for i in range(args.warmup + args.steps):
        if kind == "reference":
            if i < args.warmup:
                leaf = LEAF_SWEEP[i % len(LEAF_SWEEP)]
            else:
                leaf = min(warm, key=warm.get) if warm else None
            secs, _ = run_reference_sample(threads, leaf=leaf)
            if i < args.warmup:
                warm[leaf] = min(secs, warm.get(leaf, secs))
        else:
            secs = cpu_baseline_port(threads)
        if i >= args.warmup:
            times.append(secs)
    best_leaf = list(min(warm, key=warm.get)) if warm else None
    ms = 1000.0 * sum(times) / len(times)
    value = SAMPLE_UPDATES / (ms / 1000.0) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "GUpdates/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference init_value)", "impl": "reference",
        "config": {"workload": "jacobi2d 8192x8192 T=160 (bounded CPU sample of config 4)",
                   "parallelism": "OpenMP tasks, %d threads" % threads, "leaf": best_leaf},
        "cpu_baseline": {"value": value, "unit": "GUpdates/s", "cores": threads, "kind": kind,
                         "sample": "Jacobi-2D 8192^2 T=160, reference emitted C, leaf %s "
                                   "(fastest of the warm-up leaf sweep)" % best_leaf,
                         "host": host_info()},
        "e2e": {"value": value, "unit": "GUpdates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# BASELINE configs 0-3, reported in the same driver run as config 4 (the headline):
# (tag, kernel, params, reference CPU sample, its init-only twin, updates or flop of the sample)
PER_CONFIG = [
    ("cfg0", "jacobi2d", {"T": 256, "N": 2048}, "jacobi2d_N2048_T256", "jacobi2d_N2048_T0",
     2048 * 2048 * 256),
    ("cfg1", "heat3d_b", {"T": 100, "N": 384}, "heat3d_b_N384_T20", "heat3d_b_N384_T0", 384 ** 3 * 20),
    ("cfg2", "gs2d", {"T": 64, "N": 4096}, "gs2d_N4096_T16", "gs2d_N4096_T0", 4096 * 4096 * 16),
    ("cfg3", "gemm", {"N": 4096}, "gemm_N2048", "gemm_N1", 2 * 2048 ** 3),
]


def dmma_peak():
    """Measured fp64 DMMA peak (tools/fp64_peaks.cu on this pool's B200)."""
    try:
        with open(os.path.join(REPO, "profiles", "fp64_peaks_r01.json")) as f:
            d = json.load(f)
        return max(r["TFLOPs"] for r in d["results"] if r["probe"].startswith("dmma")), "measured"
    except (OSError, ValueError, KeyError):
        return 40.0, "fallback (nominal B200 FP64 tensor)"


def dadd_latency():
    """Measured dependent-DADD latency in cycles (tools/fp64_peaks.cu)."""
    try:
        with open(os.path.join(REPO, "profiles", "fp64_peaks_r01.json")) as f:
            for r in json.load(f)["results"]:
                if r["probe"] == "dadd_latency_cycles":
                    return float(r["value"])
    except (OSError, ValueError, KeyError):
        pass
    return 8.4


def golden_checksum(kernel, params):
    try:
        with open(os.path.join(REPO, "tests", "golden", "golden.json")) as f:
            for e in json.load(f)["entries"]:
                if e["kernel"] == kernel and e["params"] == params:
                    return e["checksum"]
    except (OSError, ValueError):
        pass
    return None


def gemm_sample_check(out, n):
    """Config 3: componentwise error on the reference's 4096 sampled cells
    (tests/golden/gemm4096_samples.json), bound 1e-12."""
    import numpy as np

    try:
        with open(os.path.join(REPO, "tests", "golden", "gemm4096_samples.json")) as f:
            g = json.load(f)
    except (OSError, ValueError):
        return {"status": "no sampled golden"}
    if g["params"]["N"] != n:
        return {"status": "sampled golden is for N=%d" % g["params"]["N"]}
    rows = np.arange(n, dtype=np.int64)
    cols = (rows * 2654435761 + 12345) % n
    got = out.reshape(n, n)[rows, cols]
    ref = np.array([int(h, 16) for h in g["out_hex"]], dtype=np.uint64).view(np.float64)
    comp = float((np.abs(got - ref) / np.array(g["absab"])).max())
    return {"cells": int(n), "componentwise_max": comp, "bound": 1e-12, "match": comp <= 1e-12,
            "exact_cells": int((got.view(np.uint64) == ref.view(np.uint64)).sum())}


def per_config(P, torch, dev, local, hbm_peak, reps_ms=1000.0):
    """BASELINE configs 0-3 through the executor's default schedule (the path a
    user of pcot::Executor gets), one GpuExecutor each."""
    import numpy as np

    flush = torch.empty(2 ** 30 // 8 * 2, dtype=torch.float64, device=dev)  # 2 GiB > L2 (126 MB)
    dpeak, dpeak_src = dmma_peak()
    res = []
    threads = os.cpu_count() or 1
    for tag, kernel, params, sample, init, sample_work in PER_CONFIG:
        with P.GpuExecutor(kernel, params, device=local) as ex:
            first = ex.run_untiled(skip_checksum=(kernel == "gemm"))
            warm = [ex.run_untiled(skip_checksum=True).device_ms for _ in range(3)]
            reps = int(max(5, min(200, reps_ms / max(min(warm), 1e-3))))
            times = []
            with ClockSampler(local) as clocks:
                for _ in range(reps):
                    flush.zero_()
                    torch.cuda.synchronize(dev)
                    times.append(ex.run_untiled(skip_checksum=True).device_ms)
            ms = statistics.median(times)
            e = {"config": tag, "kernel": kernel, "params": params, "bt": first.bt,
                 "launches_per_run": int(first.launches), "timed_runs": reps,
                 "ms_median": round(ms, 4), "ms_mean": round(statistics.mean(times), 4),
                 "ms_cov": round(statistics.pstdev(times) / statistics.mean(times), 4),
                 "l2": "2 GiB buffer written before every timed run"}
            if kernel == "gemm":
                n = params["N"]
                tf = 2.0 * n ** 3 / (ms / 1e3) / 1e12
                e["TFLOP/s"] = round(tf, 2)
                e["roofline"] = {"bound": "fp64 tensor (DMMA)", "achieved": round(tf, 2), "peak": dpeak,
                                 "unit": "TFLOP/s", "frac": round(tf / dpeak, 3), "peak_source": dpeak_src}
                e["parity"] = gemm_sample_check(ex.array_data("Out"), n)
            else:
                nd = 3 if kernel.startswith("heat3d") else 2
                upd = params["N"] ** nd * params["T"]
                gu = upd / (ms / 1e3) / 1e9
                e["GUpd/s"] = round(gu, 1)
                if kernel == "gs2d":
                    # in place: the grid crosses HBM once per launch of `seg` sweeps;
                    # the bound is the update's dependence chain, not bytes.  The
                    # wavefront h = 4t + 2i + j orders every point after all of its
                    # inputs: 4(T-1) + 3(N-3) + 1 dependent steps, each at least one
                    # update's serial latency (9 chained fp64 ops after the previous
                    # point's result + the div-by-9: 11 x the measured DADD latency)
                    fl = 11.0  # 8 DADD + div-by-9 (DMUL + 2 DFMA)
                    dadd_peak = 18.4e12  # measured DADD issue (profiles/fp64_peaks_r01.json)
                    T_, N_ = params["T"], params["N"]
                    steps = 4 * (T_ - 1) + 3 * (N_ - 3) + 1
                    lat = dadd_latency()
                    e["roofline"] = {"bound": "fp64 dependence chain (in-place wavefront)",
                                     "fp64_ops_per_update": fl,
                                     "fp64_issue_frac": round(gu * 1e9 * fl / dadd_peak, 3),
                                     "critical_path_steps": steps,
                                     "step_latency_cycles": round(fl * lat, 1),
                                     "latency_bound_ms_at_max_clock": round(steps * fl * lat / 1965e3, 4),
                                     "latency_frac": round(steps * fl * lat / 1965e3 / ms, 3),
                                     "launches_per_run": int(first.launches)}
                elif first.bt == 0:
                    # on-chip resident run (stencil2d_res.cu): the grid crosses HBM
                    # once per run (16/T B/update), so the bound is on-chip: the
                    # 5 fp64 operations per update against the measured DADD issue
                    dadd_peak = 18.4e12  # profiles/fp64_peaks_r01.json
                    e["roofline"] = {"bound": "fp64 issue (grid resident in shared memory, one launch)",
                                     "fp64_ops_per_update": 5.0, "achieved": round(gu * 5.0, 1),
                                     "peak": dadd_peak / 1e9, "unit": "Gop/s",
                                     "frac": round(gu * 5.0e9 / dadd_peak, 3),
                                     "hbm_bytes_per_update": round(16.0 / params["T"], 4)}
                else:
                    bpu = 16.0 / first.bt
                    e["roofline"] = {"bound": "hbm", "bytes_per_update": bpu, "achieved": round(gu * bpu, 1),
                                     "peak": hbm_peak, "unit": "GB/s", "frac": round(gu * bpu / hbm_peak, 3)}
                want = golden_checksum(kernel, params)
                e["parity"] = {"golden": want, "got": first.checksum_hex, "match": first.checksum_hex == want}
                if kernel.startswith("heat3d"):
                    # the next temporal depth beside the default (fewer bytes per update,
                    # lower roofline fraction): same run, same clocks, checksum-verified
                    alt = ex.run("slt", [3, 8, 8, 8])
                    ts = []
                    for _ in range(max(5, reps // 4)):
                        flush.zero_()
                        torch.cuda.synchronize(dev)
                        ts.append(ex.run("slt", [3, 8, 8, 8], skip_checksum=True).device_ms)
                    g3 = upd / (statistics.median(ts) / 1e3) / 1e9
                    e["depth_tradeoff"] = [{"bt": 3, "GUpd/s": round(g3, 1),
                                            "hbm_frac": round(g3 * 16.0 / 3 / hbm_peak, 3),
                                            "checksum_match": alt.checksum_hex == want}]
            cl = clocks.summary()
            e["clocks"] = {"sm_mhz": cl["sm_mhz"], "sm_max_mhz": cl["sm_max_mhz"], "reasons": cl["reasons"],
                           "samples": cl["samples"]}
        # the reference's own CPU path on a bounded sample of the same workload
        if os.path.exists(os.path.join(EMIT_DIR, sample)):
            secs, chk = run_reference_sample(threads, sample, init)
            unit = "GFLOP/s" if kernel == "gemm" else "GUpdates/s"
            e["cpu_baseline"] = {"value": round(sample_work / secs / 1e9, 4), "unit": unit, "cores": threads,
                                 "kind": "reference", "seconds": round(secs, 3), "checksum": chk,
                                 "sample": sample + " (reference emitted C, OpenMP, wall minus init-only run)"}
        res.append(e)
    del flush
    return res


def spawn_ranks(args):
    """`--gpus N` outside torchrun: re-launch under torch.distributed.run with
    one rank per GPU (the driver's own launch sets WORLD_SIZE and skips this)."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
           str(args.gpus), "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def dry_run(args, rank, world):
    """Rank plumbing on CPU (gloo): every rank reports in, rank 0 prints the count."""
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo")
    t = torch.ones(1)
    dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks_reporting": int(t.item()),
                          "backend": "gloo"}), flush=True)
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=32768, help="rows per rank (weak scaling)")
    ap.add_argument("--cols", type=int, default=32768)
    ap.add_argument("--T", type=int, default=512)
    ap.add_argument("--bt", type=int, default=int(os.environ.get("PCOTGPU_BT2D", 6)))
    ap.add_argument("--scheme", default="slt", choices=["slt", "cot"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--halo", default="nccl", choices=["nccl", "p2p"],
                    help="N>1 halo exchange: NCCL send/recv (overlapped) or P2P stores fused into the kernel")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-depth-sweep", action="store_true")
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="rank plumbing only (CPU, gloo)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        return spawn_ranks(args)
    rank, world, local = env_rank()
    if args.impl == "ours" and "WORLD_SIZE" in os.environ and world != args.gpus:
        sys.stderr.write("bench.py: --gpus %d but WORLD_SIZE=%d\n" % (args.gpus, world))
        return 2
    if args.dry_run:
        return dry_run(args, rank, world)

    if args.impl == "reference":
        return reference_arm(args, rank, world)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines for the driver's rank check
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")

    import torch
    import torch.distributed as dist

    import paper_1802_00166_b200 as P
    from paper_1802_00166_b200.sharded import ShardedStencil2D

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or args.halo == "p2p":
        if "MASTER_ADDR" not in os.environ:  # --halo p2p on one GPU without torchrun
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29541", RANK="0", WORLD_SIZE="1")
        dist.init_process_group("nccl", device_id=dev)
    rows = args.rows if args.scaling == "weak" else args.rows // world
    S = ShardedStencil2D(rows, args.cols, args.T, args.bt, ring_hold=0,
                         order=0 if args.scheme == "slt" else 1, device=dev, halo=args.halo)
    S.fill_init("F")
    S.snapshot_input()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        S.restart()  # every step restarts from F (copy of the step-0 slab, inside the step)
        S.run()
    barrier()
    stream = torch.cuda.current_stream(dev)
    l0 = P.lib().pcotgpu_launch_count()
    S.kernel_events.clear()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            S.restart()
            S.run(record=True)
        e1.record(stream)
        barrier()
    launches = P.lib().pcotgpu_launch_count() - l0
    ms = e0.elapsed_time(e1) / args.steps
    kms = [a.elapsed_time(b) for a, b in S.kernel_events]
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    updates = float(rows) * args.cols * args.T * world
    value = updates / (ms_max / 1e3) / 1e9

    # roofline of the dominant kernel: 16 B per cell per launch (one read + one write)
    cells = float(rows) * args.cols
    blocks = -(-args.T // args.bt)
    bytes_per_run = 16.0 * cells * blocks
    kernel_ms = sum(kms) / args.steps  # summed launch time per step
    peak, peak_src = peak_hbm()
    achieved = bytes_per_run / (kernel_ms / 1e3) / 1e9 if kernel_ms > 0 else None
    traffic = ncu_traffic(args.bt, cells) if world == 1 else None
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": (achieved / peak) if achieved else None,
            "traffic": traffic["bytes_per_launch"] if traffic else None,
            "traffic_source": traffic,
            "algorithmic_bytes_per_launch": 16.0 * cells,
            "kernel": "s2d5_kernel<bt=%d>" % args.bt, "peak_source": peak_src,
            "avg_launch_ms": (sum(kms) / len(kms)) if kms else None,
            "launches_per_step": len(kms) // max(1, args.steps),
            "bytes_per_update": 16.0 / args.bt, "kernel_share_of_step": kernel_ms / ms if ms else None,
            "dram_bytes_per_update": (traffic["bytes_per_launch"] / (cells * args.bt)) if traffic else None}

    # the same kernel at other temporal depths (one warm + one timed step
    # each, after the timed region): the throughput / HBM-fraction trade-off
    depths = []
    if world == 1 and not args.no_depth_sweep:
        for bt in (4, 5, 8):
            if bt == args.bt:
                continue
            S.bt = bt
            S.restart()
            S.run()
            S.kernel_events.clear()
            torch.cuda.synchronize()
            d0 = torch.cuda.Event(enable_timing=True)
            d1 = torch.cuda.Event(enable_timing=True)
            d0.record(stream)
            S.restart()
            S.run(record=True)
            d1.record(stream)
            torch.cuda.synchronize()
            kms_bt = sum(x.elapsed_time(y) for x, y in S.kernel_events)
            launches_bt = -(-args.T // bt)
            depths.append({"bt": bt, "GUpd/s": round(updates / (d0.elapsed_time(d1) / 1e3) / 1e9, 1),
                           "hbm_frac": round(16.0 * cells * launches_bt / (kms_bt / 1e3) / 1e9 / peak, 3)})
        S.bt = args.bt
        S.kernel_events.clear()
    roof["depth_tradeoff"] = depths

    # e2e through the C ABI with host buffers (N=1: GpuExecutor; N>1: slab copies)
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(args, P, torch, dist, S, dev, world, rows, updates, local)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(os.cpu_count() or 1)

    configs = None
    if world == 1 and not args.no_per_config:
        del S  # release config 4's slabs before the other configs allocate
        torch.cuda.empty_cache()
        configs = per_config(P, torch, dev, local, peak)

    if rank == 0:
        cl = clocks.summary()
        line = {
            "metric": METRIC, "value": value, "unit": "GUpdates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (reference init_value seeds, on device)",
            "config": {"workload": "jacobi2d (BASELINE config 4): %dx%d per rank, T=%d, zero ring"
                                   % (rows, args.cols, args.T),
                       "global_grid": [rows * world, args.cols], "T": args.T, "bt": args.bt,
                       "tile_order": args.scheme, "parallelism": "row-shard x%d" % world,
                       "halo": (None if world == 1 else
                                "NCCL send/recv of bt rows every bt steps, overlapped" if args.halo == "nccl" else
                                "P2P stores of bt rows into the neighbours' ghost rows from the stencil kernel"),
                       "l2": "inputs larger than L2 (two %.1f GiB slabs per rank)" % (cells * 8 / 2**30)},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": {"sm_mhz": cl["sm_mhz"], "sm_max_mhz": cl["sm_max_mhz"], "reasons": cl["reasons"]},
            "fp64_updates_per_step": updates,
            "per_config": configs,
        }
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0


def measure_e2e(args, P, torch, dist, S, dev, world, rows, updates, local):
    """Inputs start in pinned host memory; every step copies F in, runs, copies Out back."""
    import numpy as np

    n_cells = rows * args.cols
    # host copy of this rank's F, produced by the device generator once (untimed);
    # with several ranks on one host the output lands in a second pinned buffer
    # only at N=1 (8 ranks x 2 x 8 GiB pinned would be 128 GiB of host memory)
    host_F = torch.empty(n_cells, dtype=torch.float64, pin_memory=True)
    host_out = torch.empty(n_cells, dtype=torch.float64, pin_memory=True) if world == 1 else host_F
    stream = torch.cuda.current_stream(dev)
    if world == 1 and rows == args.cols:
        # pcotgpu_run_batch: each step's F goes in and its Out comes back through
        # pinned host memory; the copies of neighbouring steps overlap the compute
        ex = P.GpuExecutor("jacobi2d", {"T": args.T, "N": rows}, device=local)
        ex.set_stream(stream.cuda_stream)
        F_np = host_F.numpy()
        ex.array_data("F", out=F_np)
        out_np = host_out.numpy()
        sched = ("slt" if args.scheme == "slt" else "cot", [args.bt, 64, 256])
        ex.run_batch([F_np], [out_np], *sched, skip_checksum=True)  # allocates staging
        # a 64-instance batch: the first input copy and the last output copy
        # (~0.16 s each at PCIe rates) are the batch's only unoverlapped work
        steps = max(64, args.steps)
        r = ex.run_batch([F_np] * steps, [out_np] * steps, *sched, skip_checksum=True)
        ms = r.device_ms / steps
        # the batch's output equals a plain run's (first rows compared)
        ex.run(*sched, skip_checksum=True)
        ok = bool(np.array_equal(out_np[:4 * rows], ex.array_data("Out")[:4 * rows]))
        del ex
        return {"value": updates / (ms / 1e3) / 1e9, "unit": "GUpdates/s",
                "h2d_bytes_per_step": n_cells * 8, "d2h_bytes_per_step": n_cells * 8,
                "ms_per_step": ms, "steps": steps, "batch_matches_single_run": ok,
                "path": "C ABI pcotgpu_run_batch (pinned host F in, Out back, every step; "
                        "copies of adjacent steps overlap the compute)"}
    S.restart()
    host_F.copy_(S.interior(0).reshape(-1))
    torch.cuda.synchronize()

    def step():
        S.interior(0).copy_(host_F.view(rows, args.cols), non_blocking=True)
        S.exchange_sync(0)
        S.cur = 0
        S.run()
        host_out.view(rows, args.cols).copy_(S.interior(S.cur), non_blocking=True)
    step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier(device_ids=[local])
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    steps = max(1, min(args.steps, 2))
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"value": updates / (ms / 1e3) / 1e9, "unit": "GUpdates/s",
            "h2d_bytes_per_step": n_cells * 8, "d2h_bytes_per_step": n_cells * 8,
            "ms_per_step": ms, "steps": steps,
            "path": "pinned host slab copies + sharded run (per rank: the slab in, the result "
                    "back into the same pinned buffer)"}


if __name__ == "__main__":
    sys.exit(main())
