"""bench.py -- throughput of the hot path on B200 (BASELINE.json metric), one JSON line on rank 0.

A step = one pass of the whole hot path over one batch: the per-GPU shard of
BASELINE.json configs[4] (the bulk sharded run: 2^31 fp64 normals from 2^16 LFG streams
per GPU, seed 11, mu 0, sigma 1) generated once by each method B1, B2, B3 and Polar P
(seeding a1 is the one-time nrng_create, reported apart).
Weak scaling: rank r owns global streams [r 2^16, (r+1) 2^16) -- at 8 GPUs this is
exactly configs[4] (2^34 normals over 2^19 streams).  Generation needs no communication;
NCCL all-reduces only the validation moments/histograms, after the timed region.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import math
import os
import shutil
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1004_3105_b200 import workloads as W  # noqa: E402

METRIC = "fp64 normals/sec per method (B1, B3, Polar) at 1/2/4/8 B200; % of roofline"
METHODS = ("B1", "B2", "B3", "P")
CFG = W.C5_SHARD
BYTES_PER_NORMAL = 8  # algorithmic HBM traffic: one fp64 written per normal
# Algorithmic FP64 work per NORMAL, SURVEY.md §8(d) (the contract): the paper's operation tallies
# priced with CUDA libdevice fast-path DP-instruction costs.
W_SURVEY = {"B1": 34.5, "B2": 33.0, "B3": 30.5, "P": 28.5}
# The same tallies priced with this repo's own double-accurate primitives (table
# ln 8, radius from ln by one third-order rsqrt step 7, sin+cos of an exactly reduced angle 14,
# IEEE divide 8, sincos16 of P:162-170 21, Horner-15 15; MUFU seeds and integer work not
# counted), per PAIR:
#   B1 = ln + radius + sincos + 2 outputs                                   = 31
#   B2 = ln + radius + sincos16 + 2                                         = 38
#   B3 = bulk pair (m^2 1, Moebius 2, div 8, Horner 15, r 2, A 1, sincos16 21, 2) 52;
#        tail pair (1/9): 1 - m^2 1 + ln 8 + rsqrt 5 + r 2 replace 27 of it  = 52 - 11/9
#   P  = (4/pi) candidates x 3 (s) + per accepted pair ln 8 + hs 1 + rsqrt 5 + r 2 + 2 = 12/pi + 18
DP_PER_PAIR = {"B1": 31.0, "B2": 38.0, "B3": 52.0 - 11.0 / 9.0, "P": 12.0 / math.pi + 18.0}
KERNEL = {"B1": "pw_kernel<1,16>", "B2": "pw_kernel<2,16>", "B3": "b3_kernel<16>", "P": "pw_kernel<4,16>"}
FP64_PEAK_NOMINAL = 148 * 64 * 1.965e9  # SMs x FP64 lanes per SM x max SM clock = DP instr/s
# dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu --set full
# capture of the same launch (profiles/); None until captured.
TRAFFIC = {}
try:
    with open(os.path.join(ROOT, "profiles", "traffic.json")) as _fh:
        TRAFFIC = json.load(_fh)
except Exception:
    pass
# FP64 DFMA rate and HBM write bandwidth measured on this pool (tools/probe/peaks.cu: burst and
# sustained under the power cap); MEASURED_PEAKS.json (driver-written) has neither.
PROBE_PEAKS_FILE = os.path.join(ROOT, "profiles", "peaks.json")


def load_probe_peaks():
    try:
        with open(PROBE_PEAKS_FILE) as fh:
            return json.load(fh)
    except Exception:
        return None


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        # started before the warm-up (nvidia-smi takes ~0.1-0.3 s to emit its first row, longer
        # than a short timed region), line-buffered so the rows written during the timed region
        # can be told apart (mark() / stop())
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.start_row = 0
        cmd = ["nvidia-smi", "-i", str(index), "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
               "-lms", "50"]
        if shutil.which("stdbuf"):
            cmd = ["stdbuf", "-oL"] + cmd
        try:
            self.p = subprocess.Popen(cmd, stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        t0 = time.time()
        while self.p is not None and time.time() - t0 < 3.0 and not self._rows():
            time.sleep(0.02)

    def _rows(self):
        with open(self.f.name) as fh:
            return [r.split(",") for r in fh.read().strip().splitlines() if r.strip()]

    def mark(self):
        """Start of the timed region: rows before this one are the warm-up's."""
        self.start_row = len(self._rows()) if self.p is not None else 0

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.06)  # one more sampling period, so the timed region's last rows are written
        self.p.terminate()
        self.p.wait()
        allrows = self._rows()
        os.unlink(self.f.name)
        rows = allrows[self.start_row:] or allrows[-3:]  # the timed region's rows (else the last ones)
        sm = [float(r[0]) for r in rows if len(r) >= 8 and r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if len(r) >= 8 and r[1].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) < 8:
                continue
            for nm, v in zip(names, r[4:8]):
                if v.strip() == "Active":
                    reasons.add(nm)
        loaded = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": float(np.median(loaded)) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows),
                "samples_in_timed_region": len(allrows) - self.start_row}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_sample(streams_per_method: int, threads: int):
    """Time the CPU oracle, as it stands, on a bounded sample of the same workload: the first
    `streams_per_method` streams of the shard, each with the full per-stream quota
    (2^14 pairs), once per method.  Streams are independent with equal quotas, so the
    sample has the workload's exact per-stream shape."""
    import oracle as O

    O.set_threads(threads)
    per_stream = CFG.n // CFG.streams
    n = streams_per_method * per_stream
    total, secs = 0, 0.0
    per = {}
    for m in METHODS:
        st = O.Streams(CFG.seed, streams_per_method)
        t0 = time.perf_counter()
        if m == "P":
            st.normal_polar(n, CFG.mu, CFG.sigma)
        else:
            st.normal_boxmuller(n, CFG.mu, CFG.sigma, int(m[1]))
        dt = time.perf_counter() - t0
        per[m] = n / dt
        total += n
        secs += dt
    return total / secs, per, n, secs


def run_reference(args, rank):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    sample_streams = args.ref_streams
    vals = []
    for i in range(args.warmup + args.steps):
        v, per, n, secs = oracle_sample(sample_streams, threads)
        if i >= args.warmup:
            vals.append((v, per, secs))
    value = float(np.mean([v for v, _, _ in vals]))
    sample = ("%d streams x 2^14 pairs (the shard's per-stream quota) per method, %d normals per method, "
              "first streams of the seed-11 shard" % (sample_streams, sample_streams * (CFG.n // CFG.streams)))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "normals/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * float(np.mean([s for _, _, s in vals])),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(args.gpus),
        "per_method": {m: float(np.mean([p[m] for _, p, _ in vals])) for m in METHODS},
        "cpu_baseline": {"value": value, "unit": "normals/s", "cores": threads, "kind": "oracle",
                         "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "normals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def time_configs(P, torch, big, hbm_gbs, fp64_peak, sweep_calls=1000):
    """BASELINE.json configs[0..3] on this GPU, each at its own shape (one call = one batch):
    C1 B1, C2 P, C3 B2/B3, and the C4 call-length sweep (B1, P; `sweep_calls` back-to-back calls
    per length, plain and inside one CUDA graph).  Per entry: us per call, normals/s and the
    fraction of the floors -- HBM write (8 B/normal), the same plus the generator state the call
    must read and write back (floor ii), and FP64 under SURVEY 8(d)'s W."""
    res = {}
    stream = torch.cuda.current_stream()

    def timed(g, m, n, mu, sigma, calls, graph=False):
        o = big[:n]  # the caller's buffer, allocated once
        for _ in range(3):
            g.normal(m, out=o, mu=mu, sigma=sigma)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if graph:
            gr, s2 = torch.cuda.CUDAGraph(), torch.cuda.Stream()
            s2.wait_stream(stream)
            with torch.cuda.stream(s2):
                with torch.cuda.graph(gr, stream=s2):
                    for _ in range(calls):
                        g.normal(m, out=o, mu=mu, sigma=sigma)
            stream.wait_stream(s2)
            torch.cuda.synchronize()
            a.record(stream)
            gr.replay()
            b.record(stream)
        else:
            torch.cuda.synchronize()
            a.record(stream)
            for _ in range(calls):
                g.normal(m, out=o, mu=mu, sigma=sigma)
            b.record(stream)
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / calls / 1e3
        active = min(g.S, (n + 1) // 2)
        # minimal generator-state traffic per active stream: the 2 source words of each of the
        # w words it generates (at most the 607-word state) read, the last min(w, 607) written back,
        # the 8-byte counter read and written (sector granularity ignored: a lower bound)
        w = (2 if m != "B3" else 3) * ((n + 1) // 2 + g.S - 1) // g.S * (1.3 if m == "P" else 1.0)
        state = active * (8 * min(2 * w, 607) + 8 * min(w, 607) + 16)
        f_hbm = 8 * n / (hbm_gbs * 1e9)
        f_ii = (8 * n + state) / (hbm_gbs * 1e9)
        f_w = W_SURVEY[m] * n / fp64_peak
        return {"n": n, "streams": g.S, "calls": calls, "us_per_call": t * 1e6, "normals_per_s": n / t,
                "frac_hbm": f_hbm / t, "frac_floor_ii": f_ii / t, "frac_fp64_survey": f_w / t,
                "frac_roofline_i": max(f_hbm, f_w) / t, "graph": graph}

    for c in (W.C1, W.C2, W.C3):
        g = P.Generator(c.seed, c.streams)
        for m in c.methods:
            res["%s_%s" % (c.name, m)] = timed(g, m, c.n, c.mu, c.sigma, 20)
            if c.n <= (1 << 24):  # launch-latency-sized calls: also inside one CUDA graph
                res["%s_%s_graph" % (c.name, m)] = timed(g, m, c.n, c.mu, c.sigma, 20, graph=True)
        g.close()
    c = W.C4
    g = P.Generator(c.seed, c.streams)
    for m in c.methods:
        for L in W.C4_LENGTHS:
            res["C4_%s_n%d" % (m, L)] = timed(g, m, L, c.mu, c.sigma, sweep_calls)
            if L <= (1 << 18):
                res["C4_%s_n%d_graph" % (m, L)] = timed(g, m, L, c.mu, c.sigma, sweep_calls, graph=True)
    g.close()
    return res


def relaunch(n: int) -> int:
    """`python bench.py --gpus N` without a launcher: re-run this script under torchrun with
    N ranks (one per GPU, 127.0.0.1 rendezvous); rank 0's JSON line is the output."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def config_block(n_gpus):
    return {"workload": "BASELINE configs[4] per-GPU shard: 2^31 fp64 normals/GPU from 2^16 LFG(607,273) "
                        "streams/GPU (global ids [r*2^16,(r+1)*2^16)), seed 11, mu 0, sigma 1; one call per "
                        "method B1,B2,B3,P per step",
            "methods": list(METHODS), "n_per_gpu_per_method": CFG.n, "streams_per_gpu": CFG.streams,
            "seed": CFG.seed, "mu": CFG.mu, "sigma": CFG.sigma, "parallelism": "stream-sharded x%d" % n_gpus,
            "l2": "no flush needed: per call the 318 MB LFG state and 16 GiB output exceed the 126 MB L2"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ref-streams", type=int, default=4096)
    ap.add_argument("--validate", type=int, default=1)
    ap.add_argument("--configs", type=int, default=1, help="also time BASELINE configs[0..3] (N=1 only)")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(relaunch(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist

    import paper_1004_3105_b200 as P

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    t0 = time.perf_counter()
    g = P.Generator(CFG.seed, CFG.streams, first_stream=rank * CFG.streams)
    torch.cuda.synchronize()
    create_s = time.perf_counter() - t0
    out = torch.empty(CFG.n, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    def step(evs=None):
        for i, m in enumerate(METHODS):
            if evs is not None:
                evs[i][0].record(stream)
            g.normal(m, out=out, mu=CFG.mu, sigma=CFG.sigma)
            if evs is not None:
                evs[i][1].record(stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = Clocks(local)
    for _ in range(args.warmup):
        step()
    barrier()
    launches0 = g.kernel_launches
    evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in METHODS]
           for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    clocks.mark()
    start.record(stream)
    for s in range(args.steps):
        step(evs[s])
    end.record(stream)
    barrier()
    clk = clocks.stop()
    launches = g.kernel_launches - launches0
    elapsed = start.elapsed_time(end)
    per_ms = {m: float(np.mean([evs[s][i][0].elapsed_time(evs[s][i][1]) for s in range(args.steps)]))
              for i, m in enumerate(METHODS)}
    t = torch.tensor([elapsed] + [per_ms[m] for m in METHODS], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed = float(t[0])
    per_ms = {m: float(t[1 + i]) for i, m in enumerate(METHODS)}
    total_normals = world * len(METHODS) * CFG.n * args.steps
    value = total_normals / (elapsed / 1e3)

    # ---- validation: moments + histograms + serial correlation per method, all-reduced over
    # NCCL (the only exchange; dist.validate, the same code the gloo test runs on CPU)
    validation = {}
    if args.validate:
        from paper_1004_3105_b200 import dist as D

        for m in METHODS:
            g.normal(m, out=out, mu=CFG.mu, sigma=CFG.sigma)
            validation[m] = D.validate(out, CFG.n, CFG.mu, CFG.sigma, stats=P.stats, gof_hist=P.gof_hist,
                                       serial=P.serial_corr, world=world, rank=rank)

    # ---- BASELINE configs[0..3] at their own shapes (one GPU; the N>1 runs carry the shard step only)
    configs = None
    if args.configs and world == 1:
        pk = load_probe_peaks()
        configs = time_configs(P, torch, out, pk["hbm_write_gbs_sustained"] if pk else load_peaks()[0]["hbm_gbs"],
                               pk["fp64_dfma_per_s_sustained"] if pk else FP64_PEAK_NOMINAL)

    # ---- e2e: the same step through the public API with HOST output buffers (pinned),
    # the device->host copies inside the timed region (library chunked/overlapped path)
    e2e = None
    if not args.no_e2e:
        # each method's 2^31 normals go to pinned host memory through the public API; if the
        # host cannot pin 16 GiB per rank (all ranks share the node's RAM), each method's
        # batch is delivered in `parts` equal calls into a smaller buffer (same normals)
        try:
            import psutil

            avail = psutil.virtual_memory().available
        except Exception:
            avail = 64 << 30
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
        parts = 1
        while parts < 64 and CFG.n // parts * 8 * local_world > avail // 3:
            parts *= 2
        hbuf = torch.empty(CFG.n // parts, dtype=torch.float64).pin_memory()
        ge = P.Generator(CFG.seed, CFG.streams, first_stream=rank * CFG.streams)
        for m in METHODS:
            ge.normal(m, out=hbuf, mu=CFG.mu, sigma=CFG.sigma)
        barrier()
        te = time.perf_counter()
        for _ in range(args.e2e_steps):
            for m in METHODS:
                for _ in range(parts):
                    ge.normal(m, out=hbuf, mu=CFG.mu, sigma=CFG.sigma)
        barrier()
        te = torch.tensor([time.perf_counter() - te], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        ev = world * len(METHODS) * CFG.n * args.e2e_steps / float(te)
        e2e = {"value": ev, "unit": "normals/s", "h2d_bytes_per_step": 0,
               "d2h_bytes_per_step": len(METHODS) * CFG.n * 8,
               "note": "host wall clock around the host-blocking API calls, pinned host output, %d steps, "
                       "%d call(s) per method batch" % (args.e2e_steps, parts)}
        ge.close()
        del hbuf

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    peaks, peak_kind = load_peaks()
    hbm_copy = float(peaks.get("hbm_gbs", 6650.0))
    probe = load_probe_peaks()
    if probe:
        fp64_sus, fp64_burst = probe["fp64_dfma_per_s_sustained"], probe["fp64_dfma_per_s_burst"]
        hbm_w = probe["hbm_write_gbs_sustained"]
        fp64_src = "measured sustained (%s; burst %.4g)" % (os.path.relpath(PROBE_PEAKS_FILE, ROOT), fp64_burst)
        hbm_src = "measured write-only sustained (%s); MEASURED_PEAKS.json copy %.1f GB/s" % (
            os.path.relpath(PROBE_PEAKS_FILE, ROOT), hbm_copy)
    else:
        fp64_sus = fp64_burst = FP64_PEAK_NOMINAL
        hbm_w = hbm_copy
        fp64_src = "nominal 148 SMs x 64 FP64 lanes x 1965 MHz (no probe file)"
        hbm_src = peak_kind + " copy (MEASURED_PEAKS.json hbm_gbs)"
    # per method: the three floors -- HBM write (8 B/normal), FP64 under SURVEY §8(d)'s W, FP64
    # under the repo's primitive costs -- and the fraction of each; `bound_*` names the floor
    # that binds under each accounting
    per_method = {}
    for m in METHODS:
        t = per_ms[m] / 1e3
        t_hbm = BYTES_PER_NORMAL * CFG.n / (hbm_w * 1e9)
        t_w = W_SURVEY[m] * CFG.n / fp64_sus
        t_r = DP_PER_PAIR[m] * CFG.n / 2 / fp64_sus
        per_method[m] = {
            "normals_per_s": world * CFG.n / t, "ms_per_call": per_ms[m], "kernel": KERNEL[m],
            "hbm_write_gbs": BYTES_PER_NORMAL * CFG.n / t / 1e9,
            "frac_hbm": t_hbm / t, "frac_fp64_survey": t_w / t, "frac_fp64_repo": t_r / t,
            "bound_survey": "fp64" if t_w > t_hbm else "hbm", "frac_survey": max(t_w, t_hbm) / t,
            "bound_repo": "fp64" if t_r > t_hbm else "hbm", "frac_repo": max(t_r, t_hbm) / t,
            "dp_instr_per_normal_survey": W_SURVEY[m], "dp_instr_per_normal_repo": DP_PER_PAIR[m] / 2,
        }
    dom = max(METHODS, key=lambda m: per_ms[m])
    t = per_ms[dom] / 1e3
    # the dominant kernel under SURVEY §8(d) (the contract): FP64-bound for every method there
    roof = {"bound": "alu", "achieved": W_SURVEY[dom] * CFG.n / t / 1e12, "peak": fp64_sus / 1e12,
            "unit": "T DP-instr/s", "frac": W_SURVEY[dom] * CFG.n / fp64_sus / t,
            "peak_source": fp64_src, "work": "SURVEY 8(d) W_%s = %.1f DP instr/normal x %d normals per launch"
            % (dom, W_SURVEY[dom], CFG.n),
            "frac_repo_accounting": per_method[dom]["frac_repo"], "bound_repo_accounting": per_method[dom]["bound_repo"],
            "frac_burst_peak": W_SURVEY[dom] * CFG.n / fp64_burst / t,
            "hbm_peak_gbs": hbm_w, "hbm_peak_source": hbm_src,
            "kernel": "%s (%s)" % (KERNEL[dom], dom), "method": dom, "traffic": TRAFFIC.get(dom)}

    cpu = None  # the CPU oracle is timed at N = 1 only (the contract's cpu_baseline)
    if not args.no_cpu and world == 1:
        threads = os.cpu_count() or 1
        # calibrate on 256 streams, then size the sample for ~10 s of oracle wall time
        cv, _, _, csecs = oracle_sample(256, threads)
        ns = int(min(CFG.streams, max(256, 256 * 10.0 / max(csecs, 1e-3))))
        ns = min(CFG.streams, 1 << int(round(math.log2(ns))))
        cv, cper, cn, csecs = oracle_sample(ns, threads)
        # and once on a single thread, sized for ~5 s: 2^k streams x 2^14 pairs per method
        _, _, _, s1 = oracle_sample(16, 1)
        ns1 = min(CFG.streams, 1 << max(4, int(round(math.log2(16 * 5.0 / max(s1, 1e-3))))))
        v1, cper1, cn1, csecs1 = oracle_sample(ns1, 1)
        cpu = {"value": cv, "unit": "normals/s", "cores": threads, "kind": "oracle",
               "sample": "%d streams x 2^14 pairs per method (B1,B2,B3,P) = %d normals per method, %.1f s wall"
                         % (ns, cn, csecs),
               "per_method": cper, "cpu": cpu_model(),
               "single_thread": {"value": v1, "unit": "normals/s", "cores": 1, "per_method": cper1,
                                 "sample": "%d streams x 2^14 pairs per method = %d normals per method, %.1f s wall"
                                           % (ns1, cn1, csecs1)}}

    line = {
        "metric": METRIC, "value": value, "unit": "normals/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_block(world),
        "per_method": per_method,
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
        "create_s": create_s, "validation": validation, "configs": configs,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
