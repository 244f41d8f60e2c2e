#!/usr/bin/env python3
"""kog2 benchmark: 2x2 SVDs/sec (fp64 general) on B200, one JSON line.

Default workload (BASELINE.json configs[2], "cfg3"): 2^28 general fp64 2x2
matrices, entries sign * [1,2) * 2^e, e in [-500, 500], 1/8 with a random zero
pattern, generated on device by the seeded counter-based generator (SURVEY.md
§8d).  A step is one pass of the hot path — kog_svd2_batch_f64 over the batch,
inputs resident in HBM, compact results written back (96 B/matrix).  With N
GPUs (torchrun, one rank per GPU) every rank takes its own 2^28-matrix shard
of the config-5 index space (weak scaling; shard 0 is cfg3 itself) and
`value` is the whole-job rate; the fused study (generate -> svd2_ext -> svd2
-> metrics -> ErrorStats) over config 5's 2^31 matrices, combined with one
NCCL all-reduce, is reported under "study".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl kog|reference]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "2x2 SVDs/sec (fp64 general)"
UNIT = "matrices/s"
HBM_FALLBACK = 6650.0
# Reference-sequence FP64 ops per matrix (counted on the
# reference's own operation sequence by the op-counting shim, Appendix A): the
# decomposition (svd2) per config and the study (svd2 + svd2_ext + metrics).
# cfg4's count is its binary64 ops (the binary32 ones, 62, run on the FP32 pipe).
W_SVD2 = {1: 1787, 2: 88, 3: 203, 4: 328}
W_STUDY = {1: 4546, 2: 1279, 3: 1907, 4: 2803}
REF_OPS_CFG3 = W_SVD2[3]


def peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm_gbs": float(p["hbm_gbs"]), "source": "measured"}
    except Exception:
        return {"hbm_gbs": HBM_FALLBACK, "source": "fallback"}


# ------------------------------------------------------------- clocks
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    """nvidia-smi sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
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
            except Exception:
                self.proc.kill()
            if self.thread:
                self.thread.join(timeout=2)

    def summary(self) -> dict | None:
        sm, mx, reasons = [], None, set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
                mask = int(parts[2], 16) if parts[2].startswith("0x") else int(parts[2])
            except ValueError:
                continue
            mx = m
            if mask & 0x1:  # idle sample: not under load
                continue
            sm.append(s)
            for bit, name in REASONS.items():
                if mask & bit:
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def roofline(rate: float, bpm: int, w_ops: int, pk: dict, fp64_ops_s: float | None, kernel_s: float,
             traffic_bpm: float | None, kernel: str, n: int) -> dict:
    """Both bounds of one decomposition kernel: HBM (algorithmic bytes per
    matrix x rate vs the measured copy bandwidth) and FP64 (the reference's op
    count W per matrix x rate vs the in-run DFMA probe, one op per FMA); the
    binding one is the lower matrices/s."""
    achieved = bpm * rate / 1e9
    hbm_rate = pk["hbm_gbs"] * 1e9 / bpm
    out = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
           "frac": achieved / pk["hbm_gbs"], "traffic": None if traffic_bpm is None else traffic_bpm * n,
           "traffic_bytes_per_matrix": traffic_bpm, "algorithmic_bytes_per_launch": bpm * n,
           "peak_source": pk["source"], "kernel": kernel, "bytes_per_matrix": bpm, "kernel_ms": kernel_s * 1e3,
           "hbm_bound_rate": hbm_rate}
    if fp64_ops_s:
        fp_rate = fp64_ops_s / w_ops
        out.update({"fp64_ops_per_matrix": w_ops, "fp64_peak_tops": fp64_ops_s / 1e12, "fp64_bound_rate": fp_rate,
                    "fp64_achieved_tops": w_ops * rate / 1e12, "frac_fp64": rate / fp_rate,
                    "frac_hbm": achieved / pk["hbm_gbs"]})
        out["binding"] = "hbm" if hbm_rate <= fp_rate else "fp64"
        out["frac_binding"] = rate / min(hbm_rate, fp_rate)
    return out


# -------------------------------------------------------- reference arm
def run_reference(args) -> None:
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    headers compiled with the reference's Release flags) on all host cores."""
    from oracle import refbind
    from paper_2407_13116_b200 import capi, configs  # noqa: F401 (struct layouts, config)

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if not refbind.have_ref():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libkogref.so not built"}))
        return
    import numpy as np

    ref = refbind.ref()
    threads = int(ref.hardware_threads())
    cfg = configs.cfg(args.config, count=args.ref_sample).c()
    g = refbind.generate(ref, cfg, 0, cfg.count, threads=0)
    out = {k: np.empty(cfg.count, dtype=(dt or g.dtype)) for k, dt in refbind.OUT_DTYPES.items()}
    o = capi.kog_svd_out(*[out[k].ctypes.data for k in refbind.OUT_DTYPES])
    opt = capi.default_options()
    fn = ref.svd2_f32 if cfg.single_precision else ref.svd2_f64

    def step():
        fn(C.byref(refbind.mat(g)), C.byref(o), cfg.count, C.byref(opt), 0)

    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = cfg.count * args.steps / total
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32" if cfg.single_precision else "f64",
        "data": "synthetic (seeded counter-based generator, SURVEY.md §8d)",
        "config": {"workload": f"cfg{args.config} sample of {cfg.count} matrices, reference svd2 on {threads} host threads",
                   "model": "enhanced 2x2 Kogbetliantz svd2", "global_batch": cfg.count, "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "cpu_model": cpu_model(),
                         "sample": f"{cfg.count} cfg{args.config} matrices per step, std::thread over 4096-blocks"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ----------------------------------------------------------- kog2 arm
def cpu_baseline(g_host, single: bool) -> dict:
    """The reference compiled from its own headers (oracle/_ref), all host
    threads, on a bounded sample of the same workload (~10 s of wall time)."""
    from oracle import refbind
    from paper_2407_13116_b200 import capi

    if not refbind.have_ref():
        return None
    import numpy as np

    ref = refbind.ref()
    threads = int(ref.hardware_threads())
    fn = ref.svd2_f32 if single else ref.svd2_f64
    opt = capi.default_options()

    def run(n):
        g = np.ascontiguousarray(g_host[:, :n])
        out = {k: np.empty(n, dtype=(dt or g.dtype)) for k, dt in refbind.OUT_DTYPES.items()}
        o = capi.kog_svd_out(*[out[k].ctypes.data for k in refbind.OUT_DTYPES])
        t0 = time.perf_counter()
        fn(C.byref(refbind.mat(g)), C.byref(o), n, C.byref(opt), 0)
        return time.perf_counter() - t0

    n = min(1 << 22, g_host.shape[1])
    dt = run(n)
    rate = n / dt
    n2 = int(min(g_host.shape[1], max(n, rate * 8.0)))
    dt2 = run(n2)
    return {"value": n2 / dt2, "unit": UNIT, "cores": threads, "kind": "reference", "cpu_model": cpu_model(),
            "nproc": os.cpu_count(), "flags": "g++ -std=c++20 -O3 -DNDEBUG -ffp-contract=off (proj/CMakeLists.txt Release)",
            "sample": f"first {n2} matrices of the same workload, reference svd2 (oracle/_ref), "
                      f"std::thread over 4096-blocks, {dt2:.1f} s"}


def study_cpu_baseline(K) -> dict | None:
    """The reference's own run_batch (harness.hpp:226-271, threads=0 = every
    host thread; oracle/_ref) on a bounded prefix of config 5 (~8 s of wall
    time), beside the GPU study; the GPU study of the same prefix must print
    the same CSV row (csv_row, harness.hpp:275-321)."""
    from oracle import refbind
    from paper_2407_13116_b200 import configs

    if not refbind.have_ref():
        return None
    ref = refbind.ref()

    def run(n):
        c = configs.cfg(5, count=n)
        cc = c.c()
        cc.threads = 0
        t0 = time.perf_counter()
        rc, st, msg = refbind.run_batch(ref, cc)
        dt = time.perf_counter() - t0
        assert rc == 0, msg
        return dt, refbind.csv_row(ref, cc, st)

    n = 1 << 20
    dt, _ = run(n)
    n = int(min(1 << 27, max(n, (n / dt) * 8.0))) & ~4095
    dt, row = run(n)
    gpu = K.csv_row(configs.cfg(5, count=n), K.run_batch(configs.cfg(5, count=n)))
    return {"value": n / dt, "unit": UNIT, "cores": int(ref.hardware_threads()), "kind": "reference",
            "cpu_model": cpu_model(),
            "sample": f"first {n} config-5 matrices, reference run_batch (oracle/_ref, threads=0), {dt:.1f} s",
            "csv_equal": gpu == row}


def fp64_probe(K, torch) -> dict:
    """Achievable FP64 FMA rate on this GPU (DFMA chains, 8 per thread)."""
    lib = K._lib()
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    threads = sms * 2048 * 4
    iters = 4096
    sink = torch.empty(threads, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        lib.kog_fp64_probe(sink.data_ptr(), threads, iters, st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lib.kog_fp64_probe(sink.data_ptr(), threads, iters, st)
    e1.record()
    torch.cuda.synchronize()
    s = e0.elapsed_time(e1) / 1e3
    flops = threads * iters * 8 * 2
    return {"dfma_tflops": flops / s / 1e12, "fma_ops_per_s": flops / 2 / s, "sms": sms,
            "how": f"{threads} threads x {iters} x 8 independent DFMA chains"}


def time_svd2(K, torch, g, out, steps: int, warmup: int, local: int, flush=None):
    """K timed kog_svd2_batch calls over resident inputs, CUDA events on the
    launching stream around each call; with `flush` (a buffer larger than L2)
    the L2 is overwritten between calls, outside the timed events."""
    for _ in range(warmup):
        K.svd2(g, out=out)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    launches0 = K.launch_count()
    with ClockSampler(local) as clk:
        for e0, e1 in ev:
            if flush is not None:
                flush.add_(1)
            e0.record()
            K.svd2(g, out=out)
            e1.record()
        torch.cuda.synchronize()
    launches = K.launch_count() - launches0
    per = [e0.elapsed_time(e1) / 1e3 for e0, e1 in ev]
    span = ev[0][0].elapsed_time(ev[-1][1]) / 1e3
    return {"per": per, "span": span, "kernel_s": sum(per) / len(per), "launches": launches, "clocks": clk.summary()}


def load_traffic() -> dict:
    """ncu DRAM bytes per matrix of one kog_svd2_batch call per config
    (profiles/svd2_traffic.json, captured by tools/measure_traffic.sh on the
    current kernels)."""
    try:
        with open(os.path.join(ROOT, "profiles", "svd2_traffic.json")) as f:
            tr = json.load(f)
        return {int(k): v for k, v in tr.get("dram_bytes_per_matrix", {}).items()}
    except Exception:
        return {}


def l2_note(nbytes: int) -> str:
    """How the timed region relates to the 126 MB L2 (the timing rules ask for
    inputs larger than L2 or a flush between iterations)."""
    if nbytes > 4 * 126 * 2**20:
        return "inputs+outputs (%.2f GiB per GPU) larger than the 126 MB L2" % (nbytes / 2**30)
    return ("inputs+outputs (%.0f MiB per GPU) fit in the 126 MB L2: config 1 is a launch-latency-bound "
            "correctness case, not a bandwidth measurement" % (nbytes / 2**20))


SHAPE_OF = {1: "general (circ)", 2: "upper-triangular (e in [-1000,1000])", 3: "general",
            4: "general (e in [-60,60], 1% subnormal-adjacent)"}


def kernels_of(suf: str, n: int) -> str:
    """the launches behind one kog_svd2_batch call (csrc/kog2_k_svd2.cu: launch_svd2)"""
    if suf == "f64" and n >= 1 << 23:
        return ("k_svd2_lean (two-speed kernel; hands the batch back to the k_svd2_fast launched behind it if "
                "its input sample says so) + k_svd2_list (one kog_svd2_batch_f64 call)")
    return f"k_svd2_fast + k_svd2_list (one kog_svd2_batch_{suf} call)"


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kog", choices=["kog", "reference"])
    ap.add_argument("--config", type=int, default=3, choices=[1, 2, 3, 4])
    ap.add_argument("--count", type=int, default=None, help="matrices per rank (default: the config's size)")
    ap.add_argument("--ref-sample", type=int, default=1 << 24)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-study", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the cfg1/cfg2/cfg4 sub-records")
    ap.add_argument("--study-count", type=int, default=1 << 31, help="config-5 matrices over all ranks")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        run_reference(args)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2407_13116_b200 import capi, configs
    from paper_2407_13116_b200 import dist as kdist
    from paper_2407_13116_b200 import kogsvd2 as K

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())  # identity on an N-GPU box
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # nccl (one rank per GPU); KOG2_BENCH_BACKEND=gloo only for functional checks of the N>1 flow
        backend = os.environ.get("KOG2_BENCH_BACKEND", "nccl")
        dist.init_process_group(backend, device_id=dev if backend == "nccl" else None)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    capi.load()
    base = configs.cfg(5 if args.config == 3 else args.config)
    n = args.count or configs.FULL_SIZE[args.config]
    lo = rank * n  # weak scaling: rank r owns [r*n, (r+1)*n) of the config-5 index space
    g = K.generate(base, lo, n, dev)
    out = K.empty_result(n, g.dtype, dev)
    suf = "f32" if base.single_precision else "f64"
    bpm = configs.BYTES_PER_MATRIX[suf]
    torch.cuda.synchronize()

    # ---- hot path: K launches of svd2 over resident inputs (inputs > L2)
    barrier()
    torch.cuda.synchronize()
    tm = time_svd2(K, torch, g, out, args.steps, args.warmup, local)
    launches, clocks = tm["launches"], tm["clocks"]
    barrier()
    total_s = max_over_ranks(tm["span"])
    kern_s = tm["kernel_s"]
    value = world * n * args.steps / total_s
    pk = peaks()
    traffic = load_traffic()
    fp64 = fp64_probe(K, torch)
    fp64_ops = fp64["fma_ops_per_s"]
    main_roof = roofline(n / kern_s, bpm, W_SVD2[args.config], pk, fp64_ops, kern_s, traffic.get(args.config),
                         kernels_of(suf, n), n)

    # ---- the other BASELINE configs' decompositions (parity-test sizes of their own; one GPU each)
    per_config = {}
    if not args.no_configs and rank == 0 and world == 1:
        del_main = False
        for k in (1, 2, 4):
            if k == args.config:
                continue
            if not del_main:
                del g, out
                torch.cuda.empty_cache()
                del_main = True
            ck = configs.cfg(k)
            nk = configs.FULL_SIZE[k]
            sk = "f32" if ck.single_precision else "f64"
            gk = K.generate(ck, 0, nk, dev)
            ok = K.empty_result(nk, gk.dtype, dev)
            bk = configs.BYTES_PER_MATRIX[sk]
            flush = torch.empty(64 << 20, dtype=torch.int64, device=dev) if nk * bk < 4 * 126 * 2**20 else None
            tk = time_svd2(K, torch, gk, ok, max(args.steps, 10), args.warmup, local, flush)
            rk = nk / tk["kernel_s"]
            per_config[f"cfg{k}"] = {
                "workload": f"cfg{k}: {nk} {SHAPE_OF[k]} {sk} 2x2 matrices", "value": rk, "unit": UNIT,
                "ms_per_step": tk["kernel_s"] * 1e3, "steps": max(args.steps, 10), "dtype": sk,
                "l2": l2_note(nk * bk) + ("; L2 overwritten (512 MiB write) before every timed call, outside "
                                          "the timed events" if flush is not None else ""),
                "roofline": roofline(rk, bk, W_SVD2[k], pk, fp64_ops, tk["kernel_s"], traffic.get(k),
                                     kernels_of(sk, nk), nk),
                "clocks": tk["clocks"], "gpu_launches": tk["launches"]}
            del gk, ok, flush
            torch.cuda.empty_cache()
        if del_main:  # the main config's buffers back for the e2e leg below
            g = K.generate(base, lo, n, dev)
            out = K.empty_result(n, g.dtype, dev)

    # ---- fused study over config 5 with the NCCL stats all-reduce
    study = None
    if not args.no_study and args.config == 3:
        cfg5 = configs.cfg(5, count=args.study_count)
        slo, shi = kdist.shard(cfg5.count, rank, world)
        ss = K.StudyStats()
        # N>1: the stats slots all-reduced by the library's C++ side on its own NCCL
        # communicator (kog_study_allreduce); gloo runs (functional checks) use torch's
        nccl = kdist.NcclStats() if world > 1 and os.environ.get("KOG2_BENCH_BACKEND", "nccl") == "nccl" else None

        def study_step():
            ss.reset()
            ss.add(cfg5, slo, shi - slo)
            st = ss.read()
            if world == 1:
                return st
            return nccl.allreduce(st) if nccl is not None else kdist.allreduce_stats(st)

        study_step()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = study_step()
        torch.cuda.synchronize()
        dt = max_over_ranks(time.perf_counter() - t0)
        srate = cfg5.count / dt
        sbound = fp64_ops / W_STUDY[3]
        study = {"metric": "fused study matrices/s (generate+svd2+svd2_ext+metrics+reduce)",
                 "kernels": "per 2^24-matrix chunk: k_generate, k_svd2_lean + k_svd2_list, k_study_urv, "
                            "k_study_sigma, k_study_recon, k_study_ratio, k_study_ortho x2, k_study_whole, "
                            "k_study (absorb); k_study_finish once",
                 "value": srate, "unit": UNIT, "count": cfg5.count, "seconds": dt,
                 "scaling": "strong", "csv": K.csv_row(cfg5, st),
                 "allreduce": ("kog_study_allreduce (C++ ncclAllReduce MAX of the packed stats)" if nccl is not None
                               else ("torch.distributed all_reduce of the packed stats" if world > 1 else None)),
                 "roofline": {"bound": "fp64", "unit": "TOP/s", "ops_per_matrix": W_STUDY[3],
                              "achieved": W_STUDY[3] * srate / 1e12, "peak": fp64_ops / 1e12,
                              "frac": srate / sbound, "bound_rate": sbound,
                              "note": "reference-sequence FP64 ops (svd2 + svd2_ext + metrics, SURVEY.md §8(d)) "
                                      "against the in-run DFMA probe, one op per FMA; HBM is not binding "
                                      "(generated on device, 192 B/matrix of chunk buffers, ~650 B/matrix of "
                                      "DRAM traffic over the chunk's launches)"}}
        ss.free()
        if nccl is not None:
            nccl.close()

    # ---- end to end through the public host-buffer API (pinned host memory)
    e2e = None
    if not args.no_e2e:
        # host batch: the rank's whole shard at N=1; at N>1 the first 2^26 matrices of it per rank (bounds the
        # pinned host memory to 6 GiB per rank; the rate is a steady-state pipeline rate either way)
        ne = n if world == 1 else min(n, 1 << 26)
        gh = torch.empty((4, ne), dtype=g.dtype, pin_memory=True)
        gh.copy_(g[:, :ne])
        oh = {k: torch.empty(ne, dtype=v.dtype, pin_memory=True) for k, v in out.items()}
        del out
        torch.cuda.empty_cache()
        K.svd2_host(gh, out=oh)  # warm-up (pipeline buffers)
        barrier()
        steps = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(steps):
            K.svd2_host(gh, out=oh)
        dt = max_over_ranks((time.perf_counter() - t0) / steps)
        e2e = {"value": world * ne / dt, "unit": UNIT, "h2d_bytes_per_step": world * ne * (bpm - (64 if suf == "f64" else 40)),
               "d2h_bytes_per_step": world * ne * (64 if suf == "f64" else 40), "matrices_per_step": world * ne,
               "api": "kog_svd2_host_f64 (pinned host buffers, chunked H2D/kernel/D2H pipeline)"}
        g_host = gh.numpy()
    else:
        g_host = g[:, : min(n, 1 << 26)].cpu().numpy()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(g_host, base.single_precision)
        if study is not None:
            study["cpu_baseline"] = study_cpu_baseline(K)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total_s / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": suf,
            "data": "synthetic (seeded on-device counter-based generator, SURVEY.md §8d)",
            "config": {"workload": f"cfg{args.config}: {n} {SHAPE_OF[args.config]} {suf} 2x2 matrices per GPU"
                                   + (f" (e in [-500,500], 1/8 zero patterns); rank r owns indices [r*{n},(r+1)*{n}) of config 5" if args.config == 3 else ""),
                       "model": "enhanced 2x2 Kogbetliantz svd2 (arXiv 2407.13116)", "global_batch": world * n,
                       "parallelism": f"dp{world} (index-range shards, no data-path collective)",
                       "l2": l2_note(n * bpm)},
            "roofline": main_roof,
            "e2e": e2e, "cpu_baseline": cpu, "study": study, "configs": per_config or None,
            "gpu_launches": launches, "clocks": clocks, "fp64": fp64,
            "bit_exact": "outputs bit-identical to the reference (tests/test_gpu_parity.py)",
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
