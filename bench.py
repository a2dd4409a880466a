#!/usr/bin/env python
"""Benchmark: MG-Tree temporal motif co-mining on B200 (one JSON line on rank 0).

A step = one co-mining query of the configured motif group over ALL root edges of
the workload graph (window-end kernel + co-mining kernel on every rank, over a
work-balanced timestamp-range split of the roots, then one NCCL all-reduce of
the per-motif u64 counts when N > 1).  Inputs are resident in HBM; L2 (126 MB)
is flushed by a 512 MiB write between timed steps; per-step device time comes
from CUDA events on the launching stream; the job time is the max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl mayura|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Also reported: e2e (the public C-ABI path from host edge arrays: host build +
H2D + kernels + D2H of the counts), the independent per-motif GPU baseline (same
kernel, one single-motif tree per motif), roofline (algorithmic bytes of the
co-mining kernel / its event-timed duration vs measured HBM copy bandwidth),
clocks sampled during the timed region, and the CPU oracle timed on host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

KERNELS = {"flat": "co-mining pass (flat form): per MG-Tree level flat::flat_win_kernel + flat::flat_entry_kernel",
           "warp": "co-mining pass (warp form): wdfs::wdfs_kernel (warp-synchronous depth-first, lane per window entry)",
           "hybrid": "co-mining pass (hybrid form): bfs::expand_kernel + bfs::long_kernel + wdfs::wdfs_kernel"}
METRIC = "motif-group co-mining time (s) and root edges/s at 1/2/4/8 B200; HBM GB/s frac"
UNIT = "root edges/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["mayura", "reference"], default="mayura")
    ap.add_argument("--config", default="C4",
                    help="workload (synth.CONFIGS); default C4, the largest single-GPU config")
    ap.add_argument("--flush-mb", type=int, default=512)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-indep", action="store_true")
    ap.add_argument("--no-enum", action="store_true", help="skip the enumeration (NEXT-3) leg")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    ap.add_argument("--cpu-chunks", type=int, default=32, help="evenly spaced root chunks of the oracle sample")
    ap.add_argument("--profile", action="store_true", help="short run for ncu: no extras")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,utilization.gpu,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        if self.t:
            self.t.join(1)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 10:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[6:10]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ host binding --
def bind_to_gpu_numa(dev_index: int):
    """Pin this process to the CPU cores NVML reports as local to the GPU (before any pinned
    host buffer is allocated, so its pages land on the GPU's NUMA node: the e2e H2D copies then
    do not cross the socket interconnect).  Returns a record for the JSON line."""
    try:
        import pynvml
        import torch
        pr = torch.cuda.get_device_properties(dev_index)
        bus = "%08X:%02X:%02X.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        n = os.cpu_count() or 1
        mask = pynvml.nvmlDeviceGetCpuAffinity(h, (n + 63) // 64)
        cpus = {i for i in range(n) if (mask[i // 64] >> (i % 64)) & 1}
        before = len(os.sched_getaffinity(0))
        if cpus:
            os.sched_setaffinity(0, cpus)
        return {"pci_bus_id": bus, "cpus": len(cpus), "cpus_before": before}
    except Exception as e:  # no NVML / no affinity support: leave the process unbound
        return {"error": str(e)[:120]}


def unbind_all_cores():
    try:
        os.sched_setaffinity(0, set(range(os.cpu_count() or 1)))
    except Exception:
        pass


# ------------------------------------------------------------ oracle (CPU) --
def cpu_info():
    """Host CPU record for the baseline line: model, sockets, physical and logical cores."""
    rec = {"logical": os.cpu_count() or 1}
    try:
        phys, sockets, model = set(), set(), None
        cur = {}
        with open("/proc/cpuinfo") as f:
            for line in f.read().splitlines() + [""]:
                if not line.strip():
                    if cur:
                        sockets.add(cur.get("physical id", "0"))
                        phys.add((cur.get("physical id", "0"), cur.get("core id", cur.get("processor"))))
                        model = model or cur.get("model name")
                    cur = {}
                    continue
                k, _, v = line.partition(":")
                cur[k.strip()] = v.strip()
        rec.update({"model": model, "sockets": len(sockets), "physical": len(phys)})
    except OSError as e:
        rec["error"] = str(e)[:80]
    try:
        rec["affinity"] = len(os.sched_getaffinity(0))
    except Exception:
        pass
    return rec


def chunk_ranges(E: int, n_chunks: int, size: int, phase: float = 0.5):
    """n_chunks root ranges of `size` roots, evenly spaced over [0, E) (the
    oracle's C4/C5 sample is evenly spaced chunks, not one contiguous range); `phase` in [0, 1)
    places each chunk inside its stride (later waves use other phases)."""
    size = max(1, min(size, E // max(1, n_chunks)))
    if size * n_chunks >= E:
        return [(0, E)]
    stride = E / n_chunks
    return [(int(i * stride + (stride - size) * phase), int(i * stride + (stride - size) * phase) + size)
            for i in range(n_chunks)]


def describe_sample(ranges, E, n_motifs):
    if ranges == [(0, E)]:
        return "full workload (all %d roots, all %d motifs, mined independently)" % (E, n_motifs)
    n = sum(b - a for a, b in ranges)
    return ("%d evenly spaced root chunks of %d roots (%d of %d roots, %.4f%%), all %d motifs mined "
            "independently" % (len(ranges), ranges[0][1] - ranges[0][0], n, E, 100.0 * n / E, n_motifs))


def oracle_sample(E: int):
    """Root chunks of the oracle sample, in the order they are mined: the whole workload for graphs
    the oracle finishes in seconds (C1, C2), else waves of 32 evenly spaced 128-root chunks at
    shifting phases (the per-root cost is heavy-tailed, so the sample is spread over the whole
    timeline, and cut by mining time: any prefix of whole waves is itself evenly spaced)."""
    if E <= 400_000:
        return [(0, E)]
    out = []
    for ph in (0.5, 0.25, 0.75, 0.125, 0.625, 0.375, 0.875, 0.0625, 0.5625, 0.3125, 0.8125, 0.1875):
        out += chunk_ranges(E, 32, 128, ph)
    return out


def cpu_baseline(cfg, src, dst, t, V, budget_s: float, n_chunks: int = 32):
    """The oracle as it stands (O2, per-motif Algorithm 1, all host cores) on a bounded sample of the
    workload: one graph build, then the root chunks of `oracle_sample` mined until ~budget_s
    seconds of mining.  value = sampled roots / mining seconds (the build, a one-off sort and
    adjacency construction, is reported separately).  Returns (record, [(range, counts)])."""
    import oracle
    workers = os.cpu_count() or 1
    E = len(src)
    ranges = oracle_sample(E)
    per, build_s, mine_s = oracle.backtrack_ranges(src, dst, t, V, cfg.group(), cfg.delta, ranges, threads=workers,
                                                   budget_s=budget_s if len(ranges) > 1 else 0.0)
    done = ranges[:len(per)]
    rec = {"value": sum(b - a for a, b in done) / mine_s, "unit": UNIT, "cores": workers, "kind": "oracle",
           "sample": describe_sample(sorted(done), E, len(cfg.motifs)) +
                     ("" if len(ranges) == 1 else
                      "; waves of 32 evenly spaced chunks at shifting phases, mined until %.0f s" % budget_s) +
                     "; value over the mining time (graph build %.1f s not included)" % build_s,
           "seconds": mine_s, "build_seconds": build_s, "host": cpu_info()}
    return rec, list(zip(done, per))


def config_record(cfg, world, flush_mb):
    """The workload record; both arms (--impl mayura / reference) print exactly this dict."""
    gb = 96.0 * cfg.n_edges / 1e9  # device graph arrays, ~96 B per edge
    l2 = "flushed between timed steps (%d MiB write)" % flush_mb
    if gb * 1e9 > 126e6:
        l2 += "; the graph arrays (~%.1f GB) are also larger than the 126 MB L2" % gb
    return {"workload": "%s: %s" % (cfg.name, cfg.title), "name": cfg.name, "n_vertices": cfg.n_vertices,
            "n_edges": cfg.n_edges, "delta": cfg.delta, "motifs": list(cfg.motifs),
            "generator": "cascade-Zipf alpha=%g p=%g tau=%gs span=%ds seed=%d" % (
                cfg.alpha, cfg.p, cfg.tau, cfg.span, cfg.seed),
            "parallelism": "root-partition%d" % world, "l2": l2}


def run_reference(args, cfg, world, rank):
    """--impl reference: the CPU oracle as it stands (the only reference this paper-only tier
    has), on the host cores.  Each step mines the same bounded sample of the workload (the whole
    graph for C1/C2; else the evenly spaced root chunks a first pass mined in its share of ~150 s)
    over one graph build; the per-step time is the oracle's mining time.  Under torchrun only
    rank 0 runs and prints; the other ranks exit 0."""
    if rank != 0:
        return
    src, dst, t, V = cfg.graph()
    import oracle
    oracle.build()
    workers = os.cpu_count() or 1
    E = len(src)
    ranges = oracle_sample(E)
    step_budget = max(1.0, 120.0 / max(1, args.steps + args.warmup))
    if len(ranges) > 1:  # size the sample: the chunks one step's budget mines
        per, _, _ = oracle.backtrack_ranges(src, dst, t, V, cfg.group(), cfg.delta, ranges, threads=workers,
                                            budget_s=step_budget)
        ranges = ranges[:len(per)]
    reps = [ranges] * (args.warmup + args.steps)
    # all steps in one call (one graph build), each step = one pass over the sample
    per, build_s, mine_s = oracle.backtrack_ranges(src, dst, t, V, cfg.group(), cfg.delta,
                                                   [r for rep in reps for r in rep], threads=workers)
    el = mine_s * args.steps / (args.warmup + args.steps)
    n = sum(b - a for a, b in ranges)
    value = n * args.steps / el
    sample = describe_sample(sorted(ranges), E, len(cfg.motifs)) + \
        " per step; O2 per-motif Algorithm-1 backtracking; steps timed together over one graph build " \
        "(%.1f s, not included)" % build_s
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
           "data": "synthetic", "config": config_record(cfg, world, args.flush_mb),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "oracle", "sample": sample,
                            "host": cpu_info()},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def enumeration_leg(M, g, tree, cfg, src, dst, t, V, sp, stream, st, peak, got, reps: int = 3):
    """NEXT-3: mayura_enumerate into a device buffer (two kernel passes + a CUB scan + the
    tuple writes), event-timed per call on the launching stream (the call synchronises once
    in the middle to size the output).  Algorithmic bytes = 2 x the counting pass's B_alg
    (both passes traverse) + 4 B per tuple word written.  Parity vs the oracle's match lists
    (sorted per motif, every word) when the graph is small enough for the oracle."""
    import numpy as np
    import torch
    rb, re_ = 0, g.n_edges
    host_counts, need = M.mayura.mayura_enumerate_size(g.handle, tree.handle, rb, re_, sp)
    # the tuples of the whole workload may not fit next to the graph and the query scratch
    # (C4: 75 GiB): enumerate the largest centred root range whose output takes <= 60 % of free HBM
    free = torch.cuda.mem_get_info(stream.device)[0]
    while 4 * need > 0.6 * free and re_ - rb > 1000:
        n = max(1000, int((re_ - rb) * 0.6 * free / (4 * need) * 0.9))
        rb = g.n_edges // 2 - n // 2
        re_ = rb + n
        host_counts, need = M.mayura.mayura_enumerate_size(g.handle, tree.handle, rb, re_, sp)
    whole = (rb, re_) == (0, g.n_edges)
    if not whole:
        st = M.mayura_comine_stats(g.handle, tree.handle, rb, re_, False)
    buf = torch.empty(max(need, 1), dtype=torch.int32, device=stream.device)
    M.mayura_enumerate(g.handle, tree.handle, rb, re_, sp, buf, need)  # warm-up
    ms = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        c, _ = M.mayura_enumerate(g.handle, tree.handle, rb, re_, sp, buf, need)
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    t_ms = statistics.median(ms)
    matches = sum(host_counts)
    b_alg = 2 * st["bytes_alg"] + 4 * need
    parity = None
    if len(src) <= 400_000:
        import oracle
        dev_words = buf[:need].cpu().numpy().view(np.uint32)
        ok = True
        for a, mo in zip(M.split_tuples(host_counts, tree.lens, dev_words), cfg.group()):
            b = oracle.enumerate_matches(src, dst, t, V, mo, cfg.delta)
            a = np.asarray(a, np.int64)
            b = np.asarray(b, np.int64)
            if a.shape != b.shape or not np.array_equal(a[np.lexsort(a.T[::-1])], b[np.lexsort(b.T[::-1])]):
                ok = False
        parity = "exact (every tuple, sorted per motif)" if ok else "MISMATCH"
    return {"matches": matches, "words": need, "ms": t_ms, "matches_per_s": matches / (t_ms * 1e-3),
            "roots": "all" if whole else "root range [%d, %d) of %d (the whole output does not fit in free HBM)"
                                         % (rb, re_, g.n_edges),
            "counts_equal_comine": (c == got and host_counts == got) if whole else
                                   (c == host_counts == M.comine(g, tree, (rb, re_))),
            "roofline": {"bound": "hbm", "achieved": b_alg / (t_ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": b_alg / (t_ms * 1e-3) / 1e9 / peak, "bytes_alg": b_alg,
                         "note": "2 traversal passes (B_alg each) + 4 B per output word; includes the mid-call "
                                 "host sync that sizes the output"},
            "parity_vs_oracle": parity,
            "path": ("mayura_enumerate(device output), flat form: flat counting pass, then a window + entry "
                     "pass per MG-Tree level writing tuples" if M.mayura_enum_form(g.handle) == "flat" else
                     "mayura_enumerate(device output), depth-first form: per-warp count pass, CUB scan, "
                     "write pass")}


def main():
    args = parse()
    world, rank, local = dist_env()
    import synth
    cfg = synth.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg, world, rank)
        return

    import torch
    import torch.distributed as dist
    assert torch.cuda.is_available(), "bench.py needs a GPU"
    shared = os.environ.get("MAYURA_BENCH_SHARED_GPU") == "1"  # test hook: all ranks on cuda:0 over gloo
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    binding = bind_to_gpu_numa(local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    import __graft_entry__
    if rank == 0 and __graft_entry__._builder()._stale():
        __graft_entry__._builder().build()
    if world > 1:
        dist.barrier()
    import paper_2507_14813_b200 as M

    src, dst, t, V = cfg.graph()
    E = len(src)
    g = M.Graph(src, dst, t, V, device=local)
    tree = M.MGTree(cfg.group(), cfg.delta)
    k = tree.n_motifs
    from paper_2507_14813_b200 import parallel
    rb, re_ = parallel.shard_range(g, cfg.delta, rank, world)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    counts = torch.zeros(k, dtype=torch.int64, device=dev)
    flush = torch.empty(args.flush_mb * (1 << 20) // 4, dtype=torch.int32, device=dev)

    def make_events(n):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
        for e in evs:
            e.record(stream)  # materialise the cudaEvent_t before handing it to the library
        return evs

    def timed(independent: bool, steps: int, warmup: int):
        ev = [make_events(4) for _ in range(steps)]
        for i in range(warmup):
            flush.fill_(i)
            M.mayura_comine_ex(g.handle, tree.handle, rb, re_, sp, counts, independent, ev[0][1].cuda_event)
            parallel.reduce_counts(counts)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        launches0 = M.mayura_launch_count()
        for i in range(steps):
            flush.fill_(i + 1)                              # evict L2 outside the step's events
            e0, em, ek, e1 = ev[i]
            e0.record(stream)
            M.mayura_comine_ex(g.handle, tree.handle, rb, re_, sp, counts, independent, em.cuda_event)
            ek.record(stream)
            parallel.reduce_counts(counts)
            e1.record(stream)
        torch.cuda.synchronize()
        timed.launches = M.mayura_launch_count() - launches0
        if world > 1:
            dist.barrier()
        step_ms = sum(e0.elapsed_time(e1) for e0, _, _, e1 in ev)
        kern_ms = sum(em.elapsed_time(ek) for _, em, ek, _ in ev)
        win_ms = sum(e0.elapsed_time(em) for e0, em, _, _ in ev)
        tt = torch.tensor([step_ms, kern_ms, win_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return [x / steps for x in tt.tolist()], counts.cpu().tolist()

    sampler = ClockSampler(local)
    sampler.start()
    (ms_step, ms_kern, ms_win), got = timed(False, args.steps, args.warmup)
    launches = timed.launches
    clocks = sampler.stop()

    indep = None
    if not args.no_indep and not args.profile:
        (ims_step, ims_kern, _), igot = timed(True, max(3, args.steps // 2), 2)
        indep = {"ms_per_step": ims_step, "kernel_ms": ims_kern, "speedup_comine": ims_step / ms_step,
                 "counts_equal": igot == got,
                 "paper_context": "paper avg co-mining speedup 1.7x GPU (A40) / 2.4x CPU (Xeon 8380), PAPER.md:41"}

    # algorithmic bytes of the co-mining kernel for this rank's range (instrumented run, untimed)
    st = M.mayura_comine_stats(g.handle, tree.handle, rb, re_, False)
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(peaks_path):
        peak, peak_src = json.load(open(peaks_path))["hbm_gbs"], "MEASURED_PEAKS.json hbm_gbs (measured)"
    else:
        peak, peak_src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
    # SURVEY.md §8(d) B_alg: 16 B per root (src, dst, tr, hi) + 8 B per window entry + one 8-B
    # terminating entry per window; successor pointers and search probes are reported as overhead
    n_range = re_ - rb
    b_alg = 16 * n_range + 8 * (st["entries"] + st["windows"])
    achieved = b_alg / (ms_kern * 1e-3) / 1e9
    traffic, traffic_info = None, None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        tr = json.load(open(prof)).get(cfg.name)
        if tr and world == 1:
            traffic = tr.get("dram_bytes_per_launch")
            traffic_info = {"warm": tr.get("dram_bytes_per_launch_warm"), "capture": tr.get("tag"),
                            "kernels": tr.get("kernels"), "over_bytes_alg": traffic / b_alg if b_alg else None,
                            "note": "committed ncu --set full capture of one pass of this workload "
                                    "(profiles/ncu_traffic.json): cold = caches flushed before each replay, "
                                    "warm = --cache-control none"}
    form = M.mayura_kernel_form(g.handle)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_info": traffic_info,
                "kernel": KERNELS.get(form, form), "kernel_form": form,
                "kernel_ms": ms_kern,
                "window_end_kernel_ms": ms_win, "bytes_alg_per_launch": b_alg,
                "bytes_alg_per_root": b_alg / max(1, n_range),
                "bytes_alg_formula": "SURVEY.md:540 B_alg = 16*roots + 8*(window entries + windows)",
                "overhead": {"succ_ptr_bytes": 16 * st["nodes"], "search_probe_bytes_S_alg": 4 * st["probes"],
                             "impl_bytes_r1": st["bytes_alg"],
                             "note": "successor pointers (16 B per expanded node incl. the root), window-search "
                                     "probes (SURVEY.md:542 S_alg) and the r1 implementation count; frontier "
                                     "records / task stacks show in traffic"},
                "peak_source": peak_src,
                "note": "latency-bound irregular traversal; frac = algorithmic bytes / event-timed duration of "
                        "the co-mining pass (all its kernels)"}

    # e2e through the public C ABI from host buffers
    e2e = None
    if not args.no_e2e and not args.profile:
        pin_src = torch.from_numpy(src).pin_memory().numpy()
        pin_dst = torch.from_numpy(dst).pin_memory().numpy()
        pin_t = torch.from_numpy(t).pin_memory().numpy()
        tsteps = []
        for i in range(args.e2e_steps + 1):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            g2 = M.Graph(pin_src, pin_dst, pin_t, V, device=local)   # host build + H2D
            if world > 1:
                c2 = torch.zeros(k, dtype=torch.int64, device=dev)
                parallel.comine_distributed(g2, tree, c2, sp)
                host_counts = c2.cpu().tolist()                          # D2H
            else:
                host_counts = M.comine(g2, tree)                         # kernels + D2H
            g2.close()
            el = time.perf_counter() - t0
            if i > 0:
                tsteps.append(el)
            assert host_counts == got
        tt = torch.tensor([statistics.median(tsteps)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": E / tt.item(), "unit": UNIT, "s_per_step": tt.item(), "steps_s": tsteps,
               "h2d_bytes_per_step": 16 * E, "d2h_bytes_per_step": 8 * k,
               "path": "mayura_load_graph(pinned host src/dst/t -> H2D, graph build on the GPU) + "
                       "mayura_comine + D2H of the counts",
               "host_binding": binding}

    enum = None
    if world == 1 and not args.no_enum and not args.profile:
        enum = enumeration_leg(M, g, tree, cfg, src, dst, t, V, sp, stream, st, peak, got)

    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        unbind_all_cores()  # the oracle baseline uses every host core
        cpu, done = cpu_baseline(cfg, src, dst, t, V, args.cpu_budget_s)
        if [r for r, _ in done] == [(0, E)]:
            parity = "exact" if done[0][1] == got else "MISMATCH"
        else:  # every sampled chunk, per motif, vs the GPU on the same root range
            bad = [r for r, oc in done if M.comine(g, tree, r) != oc]
            parity = ("exact on all %d sampled chunks" % len(done)) if not bad else \
                     "MISMATCH on chunks %s" % bad[:8]

    if rank == 0:
        out = {"metric": METRIC, "value": E / (ms_step * 1e-3), "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
               "data": "synthetic", "config": config_record(cfg, world, args.flush_mb),
               "co_mining_time_s": ms_step * 1e-3, "counts": dict(zip(cfg.motifs, got)),
               "parity_vs_oracle": parity,
               "gpu_launches": launches * world,
               "gpu_launches_detail": "mayura_launch_count() over the timed steps x ranks: per step " +
                                      ("" if form == "flat" else "window_end_kernel + ") + KERNELS.get(form, form),
               "roofline": roofline, "clocks": clocks, "e2e": e2e, "independent_gpu": indep,
               "cpu_baseline": cpu, "search_stats": st, "enumeration": enum}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
