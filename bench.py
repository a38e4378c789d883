#!/usr/bin/env python
"""Tangram B200 load-path benchmark.

Workload (BASELINE.json configs[1]): the OPT-6.7B -> OPT-13B
model switch in a 32 GiB pool.  Loads opt13B, opt6.7B run as setup; the timed
step is the third load (opt13B again): 28 of 41 tensors reused in place
(79.4 % of 26 GB), 13 tensors (5.35 GB) placed, 18 evictions, 15 relocations
(7.62 GB compacted in 3 WAR waves), every placed and every reused tensor
content-fingerprinted.  Before each step the pool (metadata + 32 GiB arena) is
restored from a snapshot outside the timed region.

* ``value``  — effective load GB/s (model bytes / step latency) with the
  missing tensors' bytes already resident in HBM (an HBM model cache; placed
  by the K3 copy kernel): the device data plane alone.
* ``e2e``    — same metric through the C-ABI with the missing tensors in
  pinned HOST memory: H2D over PCIe inside the timed region.
* ``--impl reference`` — the reference's CPU path for the same load: the
  compiled reference's ReuseStore::load_model (oracle/_ref) plus the CPU data
  plane of apply_plan restated in oracle/cpu_oracle.c (memmove relocations,
  memcpy placements, tgfp1 fingerprints), all host threads.

Metric per step = one load.  Latency is the CUDA-event span on the pool's
stream around the synchronous tg_load_model call (host planning included);
N GPUs run N independent pools (weak scaling), max over ranks.
"""
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

GIB = 1 << 30
POOL = 32 * GIB
SEQ = ["opt13B", "opt6.7B", "opt13B"]
METRIC = "effective load GB/s, OPT-6.7B->OPT-13B switch (load #3, 79.4% tensor reuse, 32 GiB pool)"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-threads", type=int, default=0)
    p.add_argument("--profile", action="store_true", help="short run for ncu (no clocks, no baseline)")
    p.add_argument("--timeline", default="", help="write the kernel timeline of one extra value-path step "
                   "(CUPTI via torch.profiler, after the timed region) to this JSON file")
    p.add_argument("--workload", default="c2", choices=["c2", "c4"],
                   help="c2 (default): the C2 switch on every GPU; c4: GPT-20B sharded over the GPUs")
    return p.parse_args()


# ---- clocks ---------------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
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
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---- helpers -----------------------------------------------------------------------------------
def catalog(tg):
    return {m.model_id: m for m in tg.default_catalog()}


def fresh_stats(tg, upto):
    s = tg.ModelStatsTable()
    for i, mid in enumerate(SEQ[:upto]):
        s.record_request(mid, 10.0 * i)
        s.set_load_bandwidth(mid, 55e9)
    return s


def measured_h2d_peak(dev):
    """Pinned H2D bandwidth of this GPU's link (cudaMemcpyAsync, best of 3)."""
    import torch
    n = 2 * GIB
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        d.copy_(h, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    del h, d
    return n / best / 1e9


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy r+w)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---- CPU path (reference arm and cpu_baseline) ------------------------------------------------
def host_ram_gib():
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemTotal:"):
                    return round(int(ln.split()[1]) / (1 << 20), 1)
    except OSError:
        pass
    return None


def cpu_load_once(ref, cpu, rcat, arena, sources, threads):
    """The reference's CPU path for load #3: ReuseStore::load_model (compiled
    reference) + apply_plan's bytes on a host arena (oracle port), all threads.
    Returns (seconds, outcome)."""
    import numpy as np
    st = ref.ReuseStore(POOL)
    stats = ref.ModelStatsTable()
    for i, mid in enumerate(SEQ[:2]):
        stats.record_request(mid, 10.0 * i)
        stats.set_load_bandwidth(mid, 55e9)
        st.load_model(rcat[mid], stats, 10.0 * i)
        st.end_instance(mid)
    stats.record_request(SEQ[2], 20.0)
    stats.set_load_bandwidth(SEQ[2], 55e9)
    base = arena.ctypes.data
    t0 = time.perf_counter()
    o = st.load_model(rcat[SEQ[2]], stats, 20.0)
    for r in o["plan"]["relocations"]:
        cpu.copy(base + r["to"], base + r["from"], r["size"], threads)
    for p in o["plan"]["placements"]:
        cpu.copy(base + p["offset"], sources[p["tensor"]], p["size"], threads)
    final = {t["tensor"]: t for t in st.dump()["tensor_map"]}
    for t in rcat[SEQ[2]]["tensors"]:
        e = final[t["id"]]
        cpu.content_fingerprint(base + e["offset"], threads, n=e["size"])
    return time.perf_counter() - t0, o


def cpu_setup(ref, cpu, threads):
    """Host arena + host sources of load #3's misses (oracle synth)."""
    import numpy as np
    rcat = {m["model_id"]: m for m in ref.default_catalog()}
    arena = np.empty(POOL + 64, dtype=np.uint8)
    arena.fill(0)  # pre-fault
    # misses of load #3 = sources needed; find them with a dry control-plane run
    st = ref.ReuseStore(POOL)
    stats = ref.ModelStatsTable()
    for i, mid in enumerate(SEQ[:2]):
        stats.record_request(mid, 10.0 * i)
        stats.set_load_bandwidth(mid, 55e9)
        st.load_model(rcat[mid], stats, 10.0 * i)
        st.end_instance(mid)
    miss = set(st.lookup(rcat[SEQ[2]])["misses"])
    sources, keep = {}, []
    for t in rcat[SEQ[2]]["tensors"]:
        if t["id"] in miss:
            hi, lo = int(t["id"][:16], 16), int(t["id"][16:], 16)
            buf = np.empty(t["size"], dtype=np.uint8)
            cpu.synth_into(hi, lo, buf.ctypes.data, t["size"])
            keep.append(buf)
            sources[t["id"]] = buf.ctypes.data
    return rcat, arena, sources, keep


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return 0
    from oracle import cpu, ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference)"}))
        return 0
    threads = args.cpu_threads or os.cpu_count()
    rcat, arena, sources, keep = cpu_setup(ref, cpu, threads)
    total = rcat[SEQ[2]]["total_size"]
    for _ in range(args.warmup):
        cpu_load_once(ref, cpu, rcat, arena, sources, threads)
    times = []
    for _ in range(args.steps):
        s, o = cpu_load_once(ref, cpu, rcat, arena, sources, threads)
        times.append(s)
    sec = sum(times) / len(times)
    value = total / sec / 1e9
    sample = (f"load #3 of the C2 switch per step: reference ReuseStore::load_model (oracle/_ref) + CPU data plane "
              f"port (oracle/cpu_oracle.c): {len(o['plan']['relocations'])} relocations "
              f"({o['bytes_merged']} B memmove), {len(o['plan']['placements'])} placements "
              f"({o['bytes_transferred']} B memcpy from host), tgfp1 over all {len(rcat[SEQ[2]]['tensors'])} tensors "
              f"({total} B)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": "C2 OPT-6.7B->OPT-13B switch, load #3, 32 GiB pool (host arena)",
                       "threads": threads},
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": "port", "sample": sample,
                             "host_ram_gib": host_ram_gib()},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ---- ranks ----------------------------------------------------------------------------------------
def shared_gpu():
    """TANGRAM_BENCH_SHARED_GPU=1: check the N > 1 flow on a one-GPU box — every
    rank on device 0, gloo instead of NCCL (which refuses two ranks on one
    GPU), and the C2 switch shrunk to fit N copies (a flow check, not a bench
    number)."""
    return os.environ.get("TANGRAM_BENCH_SHARED_GPU") == "1"


def dist_setup():
    """(rank, world, device) from torchrun's environment; one process per GPU
    over NCCL (the barrier and the max-over-ranks reduction)."""
    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    dev = 0 if shared_gpu() else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    if world > 1:
        if shared_gpu():
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    return rank, world, dev


def reduce_max(vals, dev):
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device="cpu" if shared_gpu() else f"cuda:{dev}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


# ---- our arm ---------------------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_setup()

    import paper_2512_01357_b200 as tg
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import DeviceBuffer, PinnedBuffer
    lib = N.lib

    cat = catalog(tg)
    models = [cat[SEQ[0]], cat[SEQ[1]]]
    target = cat[SEQ[2]]

    # HBM model cache: every tensor of both models synthesised in HBM (setup
    # loads and the value path place from here).
    cache = {}
    for m in models:
        for t in m.tensors:
            if t.id not in cache:
                b = DeviceBuffer(t.size, local)
                N.check_runtime(lib.tg_synth_fill_device(t.id.c(), 0, t.size, C.c_void_p(b.ptr), local))
                cache[t.id] = b

    def register_device(ids):
        for tid in ids:
            N.check_runtime(lib.tg_host_register(tid.c(), C.c_void_p(cache[tid].ptr), cache[tid].n, None))

    register_device(cache.keys())
    pool = tg.ReuseStore(tg.GpuSpec(f"gpu{local}", POOL), device=local)
    for i, mid in enumerate(SEQ[:2]):
        st = fresh_stats(tg, i + 1)
        pool.load_model(cat[mid], st, 10.0 * i).value()
        pool.end_instance(mid)
    snap = pool.snapshot()
    hits, misses = pool.lookup(target)
    miss_ids = [t.id for t in misses]

    # pinned host copies of the misses (the e2e sources)
    host = {}
    for t in misses:
        pb = PinnedBuffer(t.size)
        N.check_runtime(lib.tg_memcpy(C.c_void_p(pb.ptr), C.c_void_p(cache[t.id].ptr), t.size))
        host[t.id] = pb

    def register_host(ids):
        for tid in ids:
            N.check_runtime(lib.tg_host_register(tid.c(), C.c_void_p(host[tid].ptr), host[tid].n, None))

    stream = torch.cuda.ExternalStream(pool.stream(), device=local)
    # default TG_LOAD_FUSED (one load-kernel launch); TANGRAM_UNFUSED=1 runs
    # the separate K3 waves + K1 passes (A/B)
    policy = tg.LoadPolicy(flags=1 | 2 | (0 if os.environ.get("TANGRAM_UNFUSED") else 8))

    def step():
        pool.restore(snap)
        st = fresh_stats(tg, 3)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        o = pool.load_model(target, st, 20.0, policy, details=False).value()
        b.record(stream)
        b.synchronize()
        return a.elapsed_time(b), o

    def phase(register):
        register(miss_ids)
        for _ in range(args.warmup):
            step()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = lib.tg_kernel_launches()
        ms, outs = [], []
        for _ in range(args.steps):
            t, o = step()
            ms.append(t)
            outs.append(o)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        launches = (lib.tg_kernel_launches() - l0) // max(1, args.steps)
        return ms, outs, launches

    clocks = ClockSampler(local)
    if not args.profile:
        clocks.start()
    ms_v, outs_v, launches = phase(register_device)
    ms_e, outs_e, _ = phase(register_host)
    clk = clocks.stop() if not args.profile else {}
    if args.timeline and rank == 0:
        write_timeline(args.timeline, lambda: (register_device(miss_ids), step()))

    def maxrank(x):
        return x if world == 1 else reduce_max([x], local)[0]

    mv = maxrank(sum(ms_v) / len(ms_v))
    me = maxrank(sum(ms_e) / len(ms_e))
    o_v, o_e = outs_v[-1], outs_e[-1]
    total = target.total_size

    # parity of the timed load (last e2e step): decisions vs the reference,
    # placed bytes vs the CPU restatement, reused bytes vs recorded digests
    parity = {"verify_mismatches": sum(o.verify_mismatches for o in outs_v + outs_e),
              "repaired_bytes": sum(o.repaired_bytes for o in outs_v + outs_e)}
    if rank == 0 and not args.profile:
        parity.update(check_parity(tg, pool, target, host, cache, local))
    kernels = isolated_kernels(tg, pool, snap, target, miss_ids, local) if not args.profile else {}

    def free_c2_working_set():
        nonlocal snap
        snap = None
        pool.close()
        for b in cache.values():
            b.free()
        for b in host.values():
            b.free()
        lib.tg_host_clear()

    c4_secondary = world > 1 and not args.profile  # the sharded + peer paths at N GPUs
    if rank != 0:
        if c4_secondary:
            free_c2_working_set()
            try:
                c4_measure(tg, rank, world, local, max(5, args.steps), max(1, min(args.warmup, 2)))
            except Exception as e:  # pragma: no cover
                print(f"rank {rank}: C4 secondary failed: {e}", file=sys.stderr)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    hbm_peak, peak_src = peaks()
    h2d_peak = measured_h2d_peak(local)
    fp_bytes = sum(t.size for t in target.tensors if t.id not in set(miss_ids))
    # K1 roofline from the e2e phase: there the reuse verification competes
    # only with the 55 GB/s H2D stream (in the value phase it shares HBM with
    # the concurrent K3 waves and placement copies, see roofline_step)
    fp_ms = statistics.mean(o.timings["fp_reuse_ms"] for o in outs_e)
    fp_ms_v = statistics.mean(o.timings["fp_reuse_ms"] for o in outs_v)
    rel_ms = statistics.mean(o.timings["relocate_ms"] for o in outs_v)
    h2d_ms = statistics.mean(o.timings["h2d_ms"] for o in outs_e)
    fp_ach = fp_bytes / (fp_ms / 1e3) / 1e9 if fp_ms > 0 else None  # fused: inside the load kernel
    rel_ach = 2 * o_v.bytes_merged / (rel_ms / 1e3) / 1e9
    h2d_ach = o_e.pcie_bytes / (h2d_ms / 1e3) / 1e9
    # minimum HBM traffic of the step: relocations r+w, placements r+w, and a
    # read of every reused tensor no copy already streams (tensors that are
    # moved or placed are fingerprinted from the copy's own read)
    # the timed loads ran with details=False: one untimed detailed replay for
    # the plan's relocation list and hit set
    pool.restore(snap)
    o_d = pool.load_model(target, fresh_stats(tg, 3), 20.0, policy).value()
    moved = {r.tensor for r in o_d.plan.relocations}
    hit_ids = set(o_d.hit_tensors)
    untouched = sum(t.size for t in target.tensors if t.id in hit_ids and t.id not in moved)
    step_bytes = 2 * o_v.bytes_merged + 2 * o_v.device_src_bytes + untouched
    step_ach = step_bytes / (mv / 1e3) / 1e9

    cpu_base = None
    extras = {}
    c4 = None
    if c4_secondary:
        free_c2_working_set()
        try:
            c4 = c4_measure(tg, rank, world, local, max(5, args.steps), max(1, min(args.warmup, 2)))
        except Exception as e:  # pragma: no cover
            c4 = {"error": f"{type(e).__name__}: {e}"}
    if not args.profile and world == 1:
        free_c2_working_set()  # before the secondary configs
        for key, fn in (("c1", lambda: run_c1(tg, local, h2d_peak, hbm_peak)), ("c3", lambda: run_c3(tg, local)),
                        ("c5", lambda: run_c5(local)),
                        ("c2_global_merge", lambda: run_c2_global_merge(tg, local, hbm_peak)),
                        ("reuse_sweep", lambda: run_reuse_sweep(tg, local, h2d_peak)),
                        ("model_store", lambda: run_model_store(tg, local, h2d_peak)),
                        ("per_model", lambda: run_per_model(tg, local, h2d_peak, hbm_peak))):
            try:  # a secondary config never takes the headline line down
                extras[key] = fn()
            except Exception as e:  # pragma: no cover
                extras[key] = {"error": f"{type(e).__name__}: {e}"}
    if not args.no_cpu_baseline and world == 1 and not args.profile:
        cpu_base = cpu_baseline(args)

    traffic = None
    tf = os.path.join(ROOT, "profiles", "load_kernel_traffic.json" if policy.flags & 8 else "fp_reuse_traffic.json")
    if os.path.exists(tf) and not shared_gpu():  # the capture is of the 32 GiB C2 step
        try:
            traffic = json.load(open(tf)).get("traffic_bytes_per_launch")
        except Exception:
            traffic = None

    fused = policy.flags & 8
    if fused:
        # the dominant (only) kernel of the step: the load kernel, timed by CUDA
        # events on the pool stream around its launch (relocate_ms), per load
        split = launches >= 2  # the load kernel + the concurrent K1 verification launch
        what = ("K3F copy_fp_kernel, the load kernel (WAR waves r+w, HBM-source placements r+w) and its "
                "concurrent K1 launch (in-place verification reads of the untouched reused tensors, taking the "
                "SM slots the load kernel releases): two launches per load, timed as one span by their "
                "globaltimer stamps (first start to last end)") if split else (
                "K3F copy_fp_kernel, the load kernel: WAR waves r+w, HBM-source placements r+w, in-place "
                "verification reads, one launch per load")
        roofline_main = {
            "bound": "hbm", "kernel": what,
            "achieved": step_bytes / (rel_ms / 1e3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
            "frac": step_bytes / (rel_ms / 1e3) / 1e9 / hbm_peak, "traffic": traffic,
            "algorithmic_bytes_per_launch": step_bytes, "ms_per_launch": rel_ms, "peak_source": peak_src}
    else:
        roofline_main = {
            "bound": "hbm", "kernel": "K1 (fingerprint-only load kernel) over the reused tensors, timed alone",
            "achieved": kernels.get("k1", {}).get("GBps"), "peak": hbm_peak, "unit": "GB/s",
            "frac": (kernels.get("k1", {}).get("GBps") or 0) / hbm_peak, "traffic": None,
            "algorithmic_bytes_per_launch": fp_bytes, "ms_per_launch": kernels.get("k1", {}).get("ms_per_launch"),
            "peak_source": peak_src, "in_step": {"GBps": fp_ach}}
    metric = METRIC if not shared_gpu() else (
        f"effective load GB/s, {SEQ[1]}->{SEQ[2]} switch (load #3, {1 - o_v.bytes_transferred / total:.1%} tensor "
        f"reuse, {POOL >> 30} GiB pool)")
    line = {
        "metric": metric,
        "value": world * total / (mv / 1e3) / 1e9,
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": mv,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic: reference catalog tensor lists, splitmix64 bytes keyed by TensorId",
        "config": {
            "workload": f"C2 switch {SEQ[0]} -> {SEQ[1]} -> {SEQ[2]}, load #3 ({SEQ[2]}) in a {POOL >> 30} GiB pool",
            "model_bytes": total, "reuse_ratio": round(1 - o_v.bytes_transferred / total, 4),
            "bytes_transferred": o_v.bytes_transferred, "bytes_merged": o_v.bytes_merged,
            "relocations": len(o_d.plan.relocations), "waves": o_v.waves, "placements": len(miss_ids),
            "reused": len(hits), "load_path": ("one load-kernel launch (TG_LOAD_FUSED)" + (
                " + a concurrent K1 launch verifying the untouched reused tensors"
                if launches >= 2 else "")) if policy.flags & 8
            else "K3 waves + K1 passes (TANGRAM_UNFUSED)",
            "value_sources": "missing tensors resident in HBM (model cache), placed by the load kernel",
            "e2e_sources": "missing tensors in pinned host memory, cudaMemcpyAsync H2D",
            "fingerprint": f"tgfp1 over all {len(target.tensors)} tensors ({len(miss_ids)} placed + {len(hits)} reused "
                           f"verified)",
            "l2": f"no flush: every step streams >= {step_bytes / 1e9:.1f} GB, >> 126 MB L2; arena restored "
                  f"(D2D {POOL // GIB} GiB) between steps",
            "timing": "CUDA events on the pool stream around each synchronous load; snapshot restore untimed; "
                      "mean over steps, max over ranks",
            "parallelism": f"{world} independent pools (one per GPU)",
        },
        "latency_ms": {"value_path": mv, "e2e": me, "plan_us": o_v.timings["plan_us"],
                       "relocate_ms": rel_ms, "h2d_ms": h2d_ms, "fp_reuse_ms_e2e": fp_ms,
                       "fp_reuse_ms_value": fp_ms_v, "fp_kernel_ms_total": o_v.timings["fp_kernel_ms"]},
        "e2e": {"value": world * total / (me / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": me,
                "h2d_bytes_per_step": o_e.pcie_bytes, "d2h_bytes_per_step": 16 * len(target.tensors)},
        "roofline": roofline_main,
        "roofline_k1": {"bound": "hbm", "kernel": f"K1 = load kernel with fingerprint-only tasks over the step's "
                                                  f"{len(hits)} reused tensors at their final offsets, one launch, "
                                                  f"timed alone",
                        "achieved": kernels.get("k1", {}).get("GBps"), "peak": hbm_peak, "unit": "GB/s",
                        "frac": (kernels.get("k1", {}).get("GBps") or 0) / hbm_peak,
                        "algorithmic_bytes_per_launch": fp_bytes,
                        "ms_per_launch": kernels.get("k1", {}).get("ms_per_launch"), "peak_source": peak_src},
        "roofline_step": {"bound": "hbm", "what": "value path: minimum device traffic of the step (relocation "
                                                  "waves r+w, HBM-source placements r+w, one read of each reused "
                                                  "tensor no copy streams) / step time",
                          "achieved": step_ach, "peak": hbm_peak, "unit": "GB/s", "frac": step_ach / hbm_peak,
                          "algorithmic_bytes_per_step": step_bytes},
        "roofline_relocate": {"bound": "hbm", "kernel": f"K3 relocate_bulk_kernel (TMA bulk copies), the step's "
                                                        f"{o_v.waves} WAR waves timed alone",
                              "achieved": kernels.get("k3", {}).get("GBps_rw"), "peak": hbm_peak, "unit": "GB/s",
                              "frac": (kernels.get("k3", {}).get("GBps_rw") or 0) / hbm_peak,
                              "algorithmic_bytes_per_load": 2 * o_v.bytes_merged,
                              "waves": kernels.get("k3", {}).get("waves"),
                              "in_step": {"GBps": rel_ach, "note": "waves overlap the K1 verification of "
                                                                   "untouched tensors"}},
        "roofline_h2d": {"bound": "pcie", "achieved": h2d_ach, "peak": h2d_peak, "unit": "GB/s",
                         "frac": h2d_ach / h2d_peak, "peak_source": "measured pinned H2D 2 GiB in this run"},
        "gpu_launches": launches,
        "clocks": clk,
        "parity": parity,
    }
    if c4 is not None:
        # N > 1: the sharded cold load (N PCIe links) and the neighbour peer
        # pull (NVLink) lead the secondary results
        line = {**{k: line[k] for k in list(line)[:12]}, "c4_sharded_and_peer": c4,
                **{k: line[k] for k in list(line)[12:]}}
        line["parity"]["c4_verify_mismatches_per_rank"] = c4.get("verify_mismatches_per_rank")
    if cpu_base:
        line["cpu_baseline"] = cpu_base
    if extras:
        line["secondary_configs"] = extras
    if shared_gpu():
        line["config"]["test_mode"] = (f"TANGRAM_BENCH_SHARED_GPU: {world} ranks on one GPU over gloo, switch "
                                       f"{SEQ} in {POOL >> 30} GiB pools — a flow check, not a bench number")
    print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def write_timeline(path, fn):
    """Kernel/memcpy start, end and stream of one step (untimed diagnostics)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    fn()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    evs = []
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        evs.append({"name": e.name[:80], "start_us": e.time_range.start, "dur_us": e.time_range.elapsed_us()})
    t0 = min((e["start_us"] for e in evs), default=0)
    for e in evs:
        e["start_us"] -= t0
    evs.sort(key=lambda e: e["start_us"])
    with open(path, "w") as f:
        json.dump(evs, f, indent=0)


def isolated_kernels(tg, pool, snap, target, miss_ids, dev, reps=5):
    """K1 and K3 timed alone on this step's own data (CUDA events around
    `reps` back-to-back launches on the launching stream):
      K1 over the 28 reused tensors at their final offsets — the same work as
         the step's reuse verification, one launch;
      K3 over each relocation wave of the step, replayed on the restored
         pre-load arena (copies are idempotent there)."""
    from paper_2512_01357_b200 import _native as N
    lib = N.lib
    miss = set(miss_ids)
    reused = [t for t in target.tensors if t.id not in miss]
    infos = [pool.tensor_info(t.id) for t in reused]
    ptrs = (C.c_void_p * len(infos))(*[i["device_ptr"] for i in infos])
    ns = (C.c_uint64 * len(infos))(*[i["size"] for i in infos])
    digs = (N.DigestC * len(infos))()
    ms = C.c_double()
    N.check_runtime(lib.tg_bench_fingerprint(ptrs, ns, len(infos), dev, reps, C.byref(ms), digs), "bench K1")
    fp_bytes = sum(i["size"] for i in infos)
    fp_ok = all((digs[k].hi, digs[k].lo) == infos[k]["digest"] for k in range(len(infos)))
    out = {"k1": {"launch_bytes": fp_bytes, "ms_per_launch": ms.value, "GBps": fp_bytes / ms.value / 1e6,
                  "digests_match_step": fp_ok}}
    # K3: plan of the step (details) on the restored arena, then each wave alone
    pool.restore(snap)
    st = fresh_stats(tg, 3)
    plan = pool.load_model(target, st, 20.0).value().plan
    pool.restore(snap)
    arena = pool.info()["arena"]
    waves = {}
    for r in plan.relocations:
        waves.setdefault(r.wave, []).append((arena + r.from_, arena + r.to, r.size))
    tot_ms, tot_bytes, per = 0.0, 0, []
    for w in sorted(waves):
        mv = waves[w]
        arr = (C.c_uint64 * (3 * len(mv)))(*[x for m in mv for x in m])
        wm = C.c_double()
        N.check_runtime(lib.tg_bench_relocate(arr, len(mv), dev, reps, C.byref(wm)), "bench K3")
        b = 2 * sum(m[2] for m in mv)
        per.append({"wave": w, "moves": len(mv), "rw_bytes": b, "ms": wm.value, "GBps_rw": b / wm.value / 1e6})
        tot_ms += wm.value
        tot_bytes += b
    out["k3"] = {"rw_bytes": tot_bytes, "ms": tot_ms, "GBps_rw": tot_bytes / tot_ms / 1e6, "waves": per}
    moved = {r.tensor for r in plan.relocations}
    out["untouched_reused_bytes"] = sum(t.size for t in reused if t.id not in moved)
    return out


_TIMER = None


def _capi_load(pool, model, stats, clock):
    """A tg_load_model call as a C/C++ host makes it: the C arguments are
    built up front and the call is timed by tools/capi_timer.cpp with CUDA
    events on the pool stream recorded in C immediately around the C-ABI
    call (host planning, launch, verification, digest readback and the
    host's post-sync bookkeeping inside; Python's ctypes overhead outside).
    Returns fn() -> (event_ms, wall_us, tg_load_outcome) (raises on error)."""
    global _TIMER
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.pool import LoadPolicy
    if _TIMER is None:
        _TIMER = C.CDLL(os.path.join(ROOT, "tools", "_build", "libcapi_timer.so"))
        _TIMER.tgt_time_load.restype = C.c_int
        _TIMER.tgt_time_load.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p,
                                         C.POINTER(C.c_double), C.POINTER(C.c_double)]
    spec, pol, out = model.c(), LoadPolicy().c(), N.LoadOutcomeC()
    ms, us = C.c_double(), C.c_double()
    h = C.cast(pool._h, C.c_void_p) if not isinstance(pool._h, int) else C.c_void_p(pool._h)
    sh = C.cast(stats._h, C.c_void_p) if not isinstance(stats._h, int) else C.c_void_p(stats._h)
    args = (h, C.cast(C.byref(spec), C.c_void_p), sh, C.c_double(clock), C.cast(C.byref(pol), C.c_void_p),
            C.cast(C.byref(out), C.c_void_p), C.byref(ms), C.byref(us))
    load = _TIMER.tgt_time_load

    def fn():
        rc = load(*args)
        if rc:
            raise RuntimeError(f"tg_load_model -> {rc}")
        return ms.value, us.value, out
    return fn


def _event_ms(stream_ptr, dev, fn):
    import torch
    s = torch.cuda.ExternalStream(stream_ptr, device=dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    r = fn()
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b), r


def run_c1(tg, dev, h2d_peak, hbm_peak, reps=3):
    """C1: OPT-1.3B cold load (PCIe) and 100 % reuse reload (HBM verify)."""
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    m = {x.model_id: x for x in tg.default_catalog()}["opt1.3B"]
    pool = tg.ReuseStore(tg.GpuSpec("gpu0", 8 * GIB), device=dev)
    cold, warm, t = [], [], 0.0
    with HostCheckpoint([m], device=dev):
        stats = tg.ModelStatsTable()
        for r in range(reps + 1):
            stats.record_request(m.model_id, t)
            ms_c, oc = _event_ms(pool.stream(), dev, lambda: pool.load_model(m, stats, t, details=False).value())
            pool.end_instance(m.model_id)
            t += 1.0
            stats.record_request(m.model_id, t)
            ms_w, _, ow = _capi_load(pool, m, stats, t)()
            pool.end_instance(m.model_id)
            pool.evict_model(m.model_id)
            t += 1.0
            if r:  # first round is warm-up
                cold.append(ms_c)
                warm.append(ms_w)
    pool.close()
    mc, mw = statistics.mean(cold), statistics.mean(warm)
    return {"workload": "C1 OPT-1.3B (2.6 GB, 25 tensors): cold load from pinned host, then 100% reuse reload "
                        "(8 GiB pool; placements identical to any larger pool)",
            "cold_ms": mc, "cold_effective_GBps": m.total_size / mc / 1e6,
            "cold_h2d_bytes": oc.pcie_bytes, "cold_h2d_ms": oc.timings["h2d_ms"],
            "warm_ms": mw, "warm_effective_GBps": m.total_size / mw / 1e6,
            "warm_fingerprint_bytes": ow.fingerprint_bytes, "warm_verify_mismatches": ow.verify_mismatches,
            "warm_device_ms": ow.total_ms, "warm_kernel_ms": ow.relocate_ms,
            "warm_timing": "CUDA events on the pool stream recorded in C immediately around one tg_load_model C-ABI "
                           "call (tools/capi_timer.cpp; arguments built beforehand): host planning, launch, "
                           "verification, digest readback and post-sync bookkeeping included",
            "plan_us_cold": oc.timings["plan_us"], "plan_us_warm": ow.plan_us,
            "cold_frac_of_h2d_peak": m.total_size / mc / 1e6 / h2d_peak,
            "warm_frac_of_hbm_peak": ow.fingerprint_bytes / mw / 1e6 / hbm_peak,
            "roofline_note": "cold: whole-load latency vs the measured pinned-H2D peak; warm: fingerprint bytes "
                             "read once / whole-load latency (plan, launch, digest readback included) vs the "
                             "measured HBM copy peak"}


def _pread_rate(path, size, threads, chunk=16 << 20):
    """GB/s of reading `size` bytes of `path` with `threads` concurrent pread
    streams of `chunk` bytes into reused buffers (the stager's read pattern
    without the copy engine)."""
    import concurrent.futures as cf
    import time
    import numpy as np
    bufs = [np.empty(chunk, np.uint8) for _ in range(threads)]
    fd = os.open(path, os.O_RDONLY)
    try:
        offs = list(range(0, size, chunk))
        def work(k):
            b = memoryview(bufs[k])
            for o in offs[k::threads]:
                n = min(chunk, size - o)
                got = 0
                while got < n:
                    r = os.preadv(fd, [b[got:n]], o + got)
                    if r <= 0:
                        raise IOError("short read")
                    got += r
        t0 = time.perf_counter()
        with cf.ThreadPoolExecutor(threads) as ex:
            list(ex.map(work, range(threads)))
        return size / (time.perf_counter() - t0) / 1e9
    finally:
        os.close(fd)


def run_model_store(tg, dev, h2d_peak, reps=3):
    """§8(f) row 2, Model Store → GPU (model.hpp:24 ModelLocation::ModelStore,
    scheduler.hpp:43-47 min(store, pcie)): OPT-6.7B written to one checkpoint
    file, every tensor registered as a file range (tg_file_register), then
    cold-loaded into an empty pool: the pool's stager threads pread 8 MiB
    chunks of every file range of the load into a 32-slot pinned ring ahead of
    the issue loop, the copy engine drains each slot into HBM as it fills, and
    the fingerprint kernels trail the copies.  Compared with the best plain
    pread rate of the same file (4..16 threads, same chunks, no copy) and the
    pinned-H2D peak: the load is bounded by min(file read, H2D)."""
    import shutil
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    m = {x.model_id: x for x in tg.default_catalog()}["opt6.7B"]
    d = os.environ.get("TANGRAM_STORE_DIR", "/tmp")
    if shutil.disk_usage(d).free < m.total_size + (4 << 30):
        return {"unavailable": f"{d}: less than {m.total_size / 1e9:.1f} GB + 4 GiB free"}
    path = os.path.join(d, f"tangram_store_{os.getpid()}.bin")
    offs = {}
    try:
        with HostCheckpoint([m], device=dev, register=False) as ck, open(path, "wb") as f:
            f.write(b"TGCK" * 3)  # odd header: file offsets of tensors unaligned, like a real checkpoint
            for t in m.tensors:
                offs[t.id] = f.tell()
                f.write(memoryview(ck.view(t.id)))
        for t in m.tensors:
            N.check_runtime(N.lib.tg_file_register(t.id.c(), path.encode(), offs[t.id], t.size, None))
        pool = tg.ReuseStore(tg.GpuSpec("gpu0", 16 * GIB), device=dev)
        stats = tg.ModelStatsTable()
        ms, fps, t = [], [], 0.0
        for r in range(reps + 1):
            stats.record_request(m.model_id, t)
            ms_l, o = _event_ms(pool.stream(), dev, lambda: pool.load_model(m, stats, t, details=False).value())
            assert o.pcie_bytes == m.total_size and o.verify_mismatches == 0
            pool.end_instance(m.model_id)
            pool.evict_model(m.model_id)
            t += 1.0
            if r:
                ms.append(ms_l)
        pool.close()
        for t_ in m.tensors:
            N.lib.tg_host_unregister(t_.id.c())
        size = os.path.getsize(path)
        pread = {n: max(_pread_rate(path, size, n) for _ in range(2)) for n in (4, 8, 12, 16)}
    finally:
        if os.path.exists(path):
            os.remove(path)
    mean = statistics.mean(ms)
    gbps = m.total_size / mean / 1e6
    threads = int(os.environ.get("TANGRAM_STAGER_THREADS", 0)) or min(16, max(4, (os.cpu_count() or 4) * 3 // 4))
    bound = min(max(pread.values()), h2d_peak)
    return {"workload": f"Model Store cold load: opt6.7B ({m.total_size / 1e9:.1f} GB, {len(m.tensors)} tensors) "
                        f"from one checkpoint file in {d} into an empty 16 GiB pool, every tensor fingerprinted",
            "load_ms": mean, "file_to_hbm_GBps": gbps,
            "stager": {"threads": threads, "chunk_MiB": 8, "ring_slots": 32},
            "pread_GBps_by_threads": pread, "file_read_GBps": max(pread.values()), "h2d_peak_GBps": h2d_peak,
            "frac_of_min_file_h2d": gbps / bound,
            "note": "page-cache state: the file was just written (hot where RAM holds it); the pread rates are "
                    "measured on the same file right after the loads, same chunking"}


def run_per_model(tg, dev, h2d_peak, hbm_peak):
    """Cold-load latency per catalog model (north star: "cold-load latency per
    model"): every default_catalog() model (catalog.hpp:72-90) loaded into an
    empty pool from pinned host memory, then reloaded at 100 % reuse (every
    tensor verified in place).  One pinned slab sized for the largest model is
    refilled per model (synthetic bytes, generated on the GPU)."""
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import DeviceBuffer, PinnedBuffer
    lib = N.lib
    models = tg.default_catalog()
    slab = PinnedBuffer(max(m.total_size for m in models))
    scratch = DeviceBuffer(max(t.size for m in models for t in m.tensors), dev)
    rows = {}
    try:
        for m in models:
            off = 0
            for t in m.tensors:
                N.check_runtime(lib.tg_synth_fill_device(t.id.c(), 0, t.size, C.c_void_p(scratch.ptr), dev))
                N.check_runtime(lib.tg_memcpy(C.c_void_p(slab.ptr + off), C.c_void_p(scratch.ptr), t.size))
                N.check_runtime(lib.tg_host_register(t.id.c(), C.c_void_p(slab.ptr + off), t.size, None))
                off += t.size
            pool = tg.ReuseStore(tg.GpuSpec("gpu0", m.total_size + (64 << 20)), device=dev)
            st = tg.ModelStatsTable()
            colds = []
            for k in range(3):  # cold = median of three loads into the emptied pool
                st.record_request(m.model_id, 0.1 * k)
                ms_c, oc = _event_ms(pool.stream(), dev, lambda: pool.load_model(m, st, 0.1 * k, details=False).value())
                pool.end_instance(m.model_id)
                colds.append(ms_c)
                if k < 2:
                    pool.evict_model(m.model_id)
            ms_c = statistics.median(colds)
            warm = []
            for k in range(4):  # the first reload is first-touch; the median of the next three is reported
                st.record_request(m.model_id, 1.0 + k)
                ms_w, _, o = _capi_load(pool, m, st, 1.0 + k)()
                warm.append((ms_w, o.relocate_ms))
                ow = {"fingerprint_bytes": o.fingerprint_bytes, "bytes_transferred": o.bytes_transferred,
                      "verify_mismatches": o.verify_mismatches}
                pool.end_instance(m.model_id)
            first_ms = warm[0][0]
            ms_w = statistics.median(w[0] for w in warm[1:])
            ow["kernel_ms"] = statistics.median(w[1] for w in warm[1:])
            pool.close()
            for t in m.tensors:
                lib.tg_host_unregister(t.id.c())
            rows[m.model_id] = {
                "bytes": m.total_size, "tensors": len(m.tensors),
                "cold_ms": ms_c, "cold_ms_each": colds, "cold_GBps": m.total_size / ms_c / 1e6,
                "cold_frac_of_h2d_peak": m.total_size / ms_c / 1e6 / h2d_peak,
                "warm_ms": ms_w, "warm_GBps": m.total_size / ms_w / 1e6,
                "warm_frac_of_hbm_peak": ow["fingerprint_bytes"] / ms_w / 1e6 / hbm_peak,
                "warm_kernel_ms": ow["kernel_ms"], "warm_first_touch_ms": first_ms,
                "warm_reuse": 1.0 - ow["bytes_transferred"] / m.total_size,
                "verify_mismatches": oc.verify_mismatches + ow["verify_mismatches"]}
    finally:
        scratch.free()
        slab.free()
    return {"workload": "every default_catalog() model: cold load into an empty pool from pinned host (PCIe; median "
                        "of three, the pool emptied between them), then a 100%-reuse reload with every tensor fingerprint-verified in place (HBM); one "
                        "CUDA-event span per synchronous load; warm: events recorded in C around the C-ABI call "
                        "(tools/capi_timer.cpp), median of 3 reloads after a first-touch one (reported too)", "models": rows}


def run_c2_global_merge(tg, dev, hbm_peak, reps=3):
    """C2's compaction stress case: the same switch under
    LoadPolicy{merge=GlobalMerge} in a 36 GiB pool — load #3 relocates 13
    tensors in 11 serial WAR waves, all gated inside one load-kernel launch.
    HBM-resident sources, pool restored from a snapshot before each rep."""
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import DeviceBuffer
    lib = N.lib
    cat = catalog(tg)
    seq = ["opt13B", "opt6.7B", "opt13B"]
    bufs = []
    for mid in seq[:2]:
        for t in cat[mid].tensors:
            b = DeviceBuffer(t.size, dev)
            N.check_runtime(lib.tg_synth_fill_device(t.id.c(), 0, t.size, C.c_void_p(b.ptr), dev))
            N.check_runtime(lib.tg_host_register(t.id.c(), C.c_void_p(b.ptr), t.size, None))
            bufs.append((t.id, b))
    pool = tg.ReuseStore(tg.GpuSpec("gpu0", 36 * GIB), device=dev)
    policy = tg.LoadPolicy(merge=1, flags=1 | 2 | 8)

    def stats(upto):
        s = tg.ModelStatsTable()
        for i, mid in enumerate(seq[:upto]):
            s.record_request(mid, 10.0 * i)
            s.set_load_bandwidth(mid, 55e9)
        return s
    try:
        for i, mid in enumerate(seq[:2]):
            pool.load_model(cat[mid], stats(i + 1), 10.0 * i, policy).value()
            pool.end_instance(mid)
        snap = pool.snapshot()
        ms, kms, o = [], [], None
        for r in range(reps + 1):
            pool.restore(snap)
            t, o = _event_ms(pool.stream(), dev, lambda: pool.load_model(cat[seq[2]], stats(3), 20.0, policy,
                                                                          details=(r == 0)).value())
            if r == 0:
                plan = o.plan
                continue
            ms.append(t)
            kms.append(o.timings["relocate_ms"])
        snap = None
        m, k = statistics.mean(ms), statistics.mean(kms)
        moved = {x.tensor for x in plan.relocations}
        untouched = sum(t.size for t in cat[seq[2]].tensors if t.id not in moved) - o.bytes_transferred
        algo = 2 * o.bytes_merged + 2 * o.device_src_bytes + untouched
        return {"workload": "C2 switch under GlobalMerge, 36 GiB pool, load #3 (opt13B), HBM sources",
                "relocations": len(plan.relocations), "waves": o.waves, "bytes_merged": o.bytes_merged,
                "bytes_transferred": o.bytes_transferred, "ms": m, "effective_GBps": cat[seq[2]].total_size / m / 1e6,
                "load_kernel_ms": k, "load_kernel_GBps": algo / k / 1e6, "load_kernel_frac_of_hbm_peak":
                    algo / k / 1e6 / hbm_peak, "algorithmic_bytes": algo,
                "verify_mismatches": o.verify_mismatches}
    finally:
        pool.close()
        for tid, b in bufs:
            lib.tg_host_unregister(tid.c())
            b.free()


def run_reuse_sweep(tg, dev, h2d_peak=None, reps=3):
    """Effective load GB/s at stated reuse ratios (north star): the C2 switch's
    load #3 in 30 / 32 / 36 / 40 GiB pools (reuse 71.5 / 79.4 / 96.8 / 100 %),
    value path (misses from the HBM cache) and e2e (misses from pinned host
    memory over PCIe), pool restored from a snapshot before each rep."""
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import DeviceBuffer, PinnedBuffer
    lib = N.lib
    cat = catalog(tg)
    seq = ["opt13B", "opt6.7B", "opt13B"]
    target = cat[seq[2]]
    cache = {}
    for mid in seq[:2]:
        for t in cat[mid].tensors:
            b = DeviceBuffer(t.size, dev)
            N.check_runtime(lib.tg_synth_fill_device(t.id.c(), 0, t.size, C.c_void_p(b.ptr), dev))
            cache[t.id] = b

    def register(tids, src):
        for tid in tids:
            N.check_runtime(lib.tg_host_register(tid.c(), C.c_void_p(src[tid].ptr), src[tid].n, None))

    def stats(upto):
        s = tg.ModelStatsTable()
        for i, mid in enumerate(seq[:upto]):
            s.record_request(mid, 10.0 * i)
            s.set_load_bandwidth(mid, 55e9)
        return s
    rows = {}
    try:
        for gib in (30, 32, 36, 40):
            register(cache.keys(), cache)
            pool = tg.ReuseStore(tg.GpuSpec("gpu0", gib * GIB), device=dev)
            for i, mid in enumerate(seq[:2]):
                pool.load_model(cat[mid], stats(i + 1), 10.0 * i).value()
                pool.end_instance(mid)
            snap = pool.snapshot()
            _, misses = pool.lookup(target)
            host = {}
            for t in misses:
                pb = PinnedBuffer(t.size)
                N.check_runtime(lib.tg_memcpy(C.c_void_p(pb.ptr), C.c_void_p(cache[t.id].ptr), t.size))
                host[t.id] = pb
            out = {}
            for name, src in (("value", cache), ("e2e", host)):
                register([t.id for t in misses], src)
                ms = []
                for r in range(reps + 1):
                    pool.restore(snap)
                    t, o = _event_ms(pool.stream(), dev, lambda: pool.load_model(target, stats(3), 20.0,
                                                                                  details=False).value())
                    if r:
                        ms.append(t)
                m = statistics.mean(ms)
                tl = o.timings
                out[name] = {"ms": m, "effective_GBps": target.total_size / m / 1e6,
                             # device timeline of the last rep, from entry: the load kernel ends; the first
                             # H2D gated on a relocation wave may start (cuStreamWaitValue64 on the wave's
                             # tile counter, before the kernel ends); the H2D span
                             "timeline_ms": {"kernel_end": tl["kernel_end_ms"],
                                             "gated_h2d_start": tl["gated_h2d_start_ms"],
                                             "h2d_span": tl["h2d_ms"], "total": tl["total_ms"]}}
                if name == "e2e" and o.pcie_bytes and h2d_peak:
                    # the load's floor: its missed bytes over the measured pinned-H2D link
                    out[name]["pcie_floor_ms"] = o.pcie_bytes / h2d_peak / 1e6
                    out[name]["frac_of_pcie_floor"] = out[name]["pcie_floor_ms"] / m
                assert o.verify_mismatches == 0
            rows[f"{gib}GiB"] = {"reuse_ratio": 1.0 - o.bytes_transferred / target.total_size,
                                 "bytes_transferred": o.bytes_transferred, "bytes_merged": o.bytes_merged,
                                 **out}
            snap = None
            pool.close()
            for b in host.values():
                b.free()
            lib.tg_host_clear()
    finally:
        lib.tg_host_clear()
        for b in cache.values():
            b.free()
    return {"workload": "C2 switch load #3 (opt13B after opt13B, opt6.7B) at four pool sizes; value = misses "
                        "from an HBM cache (load kernel), e2e = misses from pinned host memory (PCIe)",
            "pools": rows}


def run_c3(tg, dev):
    """C3: Llama-2-13B load + on-demand KV block allocation under a prefill
    burst (16 / 64 ShareGPT prompts, seed 7 — the golden request lists) and one
    decode-step batch; device block tables; vs the reference KvEngine."""
    import time
    import torch
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import DeviceBuffer
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", "c3_kv.json")))
    model = tg.make_model("llama2-13B", 26_000_000_000, 40, 819_200)
    bufs = []
    for t in model.tensors:
        b = DeviceBuffer(t.size, dev)
        N.lib.tg_synth_fill_device(t.id.c(), 0, t.size, C.c_void_p(b.ptr), dev)
        N.lib.tg_host_register(t.id.c(), C.c_void_p(b.ptr), t.size, None)
        bufs.append(b)
    pool = tg.ReuseStore(tg.GpuSpec("gpu0", 120 * GIB), device=dev)
    stats = tg.ModelStatsTable()
    stats.record_request(model.model_id, 0.0)
    pool.load_model(model, stats, 0.0).value()
    for b in bufs:
        b.free()
    N.lib.tg_host_clear()
    out = {}
    try:
        from oracle import ref
        have_ref = ref.available()
    except Exception:
        have_ref = False
    for n, case in golden.items():
        reqs = [tuple(r) for r in case["requests"]]
        dec = [(r, (p + 15) // 16 * 16 + 1) for r, p in reqs]
        kv = tg.KvEngine("llama2-13B", 16, 819_200)
        kv.batch_allocate(pool, stats, reqs, want_pbns=False)  # warm-up (device arrays sized)
        kv.instance_teardown(pool)
        best_b, best_d, counts = 1e9, 1e9, None
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            counts = kv.batch_allocate(pool, stats, reqs, want_pbns=False).value()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            kv.batch_allocate(pool, stats, dec, want_pbns=False).value()
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            best_b, best_d = min(best_b, t1 - t0), min(best_d, t2 - t1)
            kv.instance_teardown(pool)
        blocks = sum(counts)
        row = {"requests": len(reqs), "blocks": blocks, "blocks_match_reference": blocks == sum(
                   len(g) for g in case["burst"]),
               "burst_us": best_b * 1e6, "decode_step_us": best_d * 1e6, "blocks_per_us": blocks / (best_b * 1e6)}
        # K4D: decode steps decided on the device (no host round trip per
        # step): S steps in which every request crosses a block boundary
        kv.batch_allocate(pool, stats, reqs, want_pbns=False).value()
        steps = 8
        slots = torch.tensor([kv.request_slot(r) for r, _ in reqs], dtype=torch.int64, device=f"cuda:{dev}")
        same = torch.tensor([p for _, p in reqs], dtype=torch.int64, device=f"cuda:{dev}")
        kv.device_arm(pool, 8192 // 16 + steps + 2, len(reqs), 1).value()  # warm-up: a no-grant batch
        kv.batch_allocate_device(slots.data_ptr(), same.data_ptr(), len(reqs))
        kv.device_sync(pool, stats).value()
        kv.device_arm(pool, 8192 // 16 + steps + 2, len(reqs), steps).value()
        toks = [torch.tensor([(p + 15) // 16 * 16 + 1 + 16 * k for _, p in reqs], dtype=torch.int64,
                             device=f"cuda:{dev}") for k in range(steps)]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cs = torch.cuda.current_stream()
        e0.record(cs)
        for k in range(steps):
            kv.batch_allocate_device(slots.data_ptr(), toks[k].data_ptr(), len(reqs), stream=cs.cuda_stream)
        e1.record(cs)
        torch.cuda.synchronize()
        applied, replayed = kv.device_sync(pool, stats).value()
        want_blocks = sum(((p + 15) // 16 * 16 + 1 + 16 * (steps - 1) + 15) // 16 for _, p in reqs)
        row["device_decode_step_us"] = e0.elapsed_time(e1) * 1e3 / steps
        row["device_decode_steps"] = steps
        row["device_steps_applied_on_device"] = applied
        row["device_blocks_match"] = sum(kv._blocks(r) for r, _ in reqs) == want_blocks
        kv.instance_teardown(pool)
        if have_ref:
            r = ref.ReuseStore(120 * GIB)
            rs = ref.ModelStatsTable()
            rs.record_request(model.model_id, 0.0)
            r.load_model(model.to_json(), rs, 0.0)
            rk = ref.KvEngine("llama2-13B", 16, 819_200)
            rb = rk.batch_allocate(r, rs, reqs)
            rd = rk.batch_allocate(r, rs, dec)
            row["reference_cpu_burst_us"] = rb["ns"] / 1e3
            row["reference_cpu_decode_step_us"] = rd["ns"] / 1e3
        out[n] = row
    pool.close()
    return {"workload": "C3 Llama-2-13B (26 GB) in a 120 GiB pool; KV blocks of 16 tokens x 819,200 B/token; "
                        "host+device time per batch incl. kernel completion, best of 3; device_decode_step_us: "
                        "K4D batches decided on the GPU (tg_kv_batch_allocate_device), CUDA-event time per step "
                        "over 8 back-to-back steps in which every request crosses a block boundary",
            "bursts": out}


def _replay(bin_, args, env, timeout=900):
    """One simulator run: (stdout bytes, the binding's stderr report or None, rc)."""
    r = subprocess.run([bin_] + args, capture_output=True, timeout=timeout, env=env)
    rep = None
    try:
        rep = json.loads(r.stderr.decode().strip().splitlines()[-1])
    except Exception:
        pass
    return r.stdout, rep, r.returncode


C5_REAL_MODELS = ["opt1.3B", "qwen3B", "llama3B", "opt6.7B", "llama8B", "yi9B"]


def run_c5(dev):
    """C5: the reference's own Simulator (unmodified
    simulator.hpp) replays Zipf traces over the drop-in bindings.

    * full: the C5 config (8 x 48 GiB, 2,000 requests) with asynchronous loads
      (TG_LOAD_ASYNC); pool gpuK lives on CUDA device K when it exists (so on
      an 8-GPU box every pool moves real bytes and loads overlap across GPUs),
      else control-plane only; sources synthesised in HBM on device 0.
      RunMetrics must equal the pure-reference build's.
    * real4: every pool real — 4 x 24 GiB pools on this GPU (one per GPU where
      4 exist), the six smallest catalog models (62 GB, so models migrate
      between pools), sources in pinned host memory: synchronous loads,
      asynchronous loads (both byte-identical RunMetrics to the reference),
      and the peer-aware schedule (TANGRAM_PEER_SCHEDULE: misses resident on
      another pool come over NVLink / the SM copy instead of PCIe; decisions
      differ from the reference's by design)."""
    import time
    import torch
    build = os.path.join(ROOT, "integration", "_build")
    ref_bin, tg_bin = os.path.join(build, "sim_reference"), os.path.join(build, "sim_tangram")
    if not (os.path.exists(ref_bin) and os.path.exists(tg_bin)):
        return {"unavailable": "integration/_build binaries absent (built by build() where the reference exists)"}
    out = {}
    args = ["reuse_odkv", "8", "48", "4", "2", "2000", "42", "0", "0", "L3"]
    ref_out = subprocess.run([ref_bin] + args, capture_output=True, timeout=600).stdout
    env = dict(os.environ, TANGRAM_DEVICE="auto", TANGRAM_SYNTH_SOURCES="1", TANGRAM_ASYNC_LOADS="1")
    t0 = time.perf_counter()
    b_out, rep, rc = _replay(tg_bin, args, env)
    wall = time.perf_counter() - t0
    if rep is None:
        return {"unavailable": f"replay failed rc={rc}"}
    real = [p for p in rep["pools"] if p["device"] >= 0]
    moved = sum(p["relocated_bytes"] + p["device_src_bytes"] + p["pcie_bytes"] + p["peer_bytes"] for p in real)
    out["full"] = {
        "workload": "C5 Zipf trace (2,000 requests, seed 42, L3) on 8 x 48 GiB pools, ReuseOdkv, batch 4, "
                    "keep-alive 2 s; reference Simulator over the drop-in bindings, asynchronous loads; pools on "
                    f"devices: {[p['gpu_id'] for p in real]} (the rest control-plane only), HBM-resident sources",
        "run_metrics_equal_reference": rc == 0 and b_out == ref_out,
        "pools_with_bytes": len(real),
        "loads": sum(p["loads"] for p in real),
        "moved_bytes": moved,
        "fingerprint_bytes": sum(p["fingerprint_bytes"] for p in real),
        "verify_mismatches": sum(p["verify_mismatches"] for p in real),
        "failed_loads": sum(p["failed_loads"] for p in real),
        "data_plane_ms_per_pool": {p["gpu_id"]: p["data_plane_ms"] for p in real},
        "replay_run_s": rep.get("run_s"), "replay_wall_s": wall}
    ngpu = torch.cuda.device_count()
    args4 = ["reuse_odkv", "4", "24", "4", "2", "400", "42", "0", "0", "L3", ",".join(C5_REAL_MODELS)]
    ref4 = subprocess.run([ref_bin] + args4, capture_output=True, timeout=600).stdout
    base_env = dict(os.environ, TANGRAM_SYNTH_SOURCES="host", TANGRAM_DEVICE="auto" if ngpu >= 4 else "0")
    modes = {}
    for name, extra in (("sync", {"TANGRAM_ASYNC_LOADS": "0"}), ("async", {"TANGRAM_ASYNC_LOADS": "1"}),
                        ("peer", {"TANGRAM_ASYNC_LOADS": "1", "TANGRAM_PEER_SCHEDULE": "700"})):
        o, r, rc = _replay(tg_bin, args4, dict(base_env, **extra))
        if r is None:
            modes[name] = {"error": f"rc={rc}"}
            continue
        pools = r["pools"]
        pcie = sum(p["pcie_bytes"] for p in pools)
        peer = sum(p["peer_bytes"] for p in pools)
        dp = sum(p["pcie_bytes"] + p["peer_bytes"] + p["device_src_bytes"] + p["relocated_bytes"] for p in pools)
        modes[name] = {
            "run_metrics_equal_reference": rc == 0 and o == ref4,
            "loads": sum(p["loads"] for p in pools), "pcie_bytes": pcie, "peer_bytes": peer,
            "fingerprint_bytes": sum(p["fingerprint_bytes"] for p in pools),
            "verify_mismatches": sum(p["verify_mismatches"] for p in pools),
            "failed_loads": sum(p["failed_loads"] for p in pools),
            "replay_run_s": r.get("run_s"), "replay_s": r.get("replay_s"),
            "data_plane_ms_sum": sum(p["data_plane_ms"] for p in pools),
            "placed_GBps_over_run": (pcie + peer) / r["run_s"] / 1e9 if r.get("run_s") else None,
            "data_plane_GBps_over_run": dp / r["run_s"] / 1e9 if r.get("run_s") else None}
    if "pcie_bytes" in modes.get("peer", {}) and "pcie_bytes" in modes.get("sync", {}):
        modes["peer"]["pcie_bytes_saved_vs_reference_schedule"] = modes["sync"]["pcie_bytes"] - modes["peer"]["pcie_bytes"]
    out["real4"] = {
        "workload": "C5-shaped replay, every pool with real bytes: 4 x 24 GiB pools, models "
                    f"{','.join(C5_REAL_MODELS)} (62 GB), 400 requests, seed 42, L3, ReuseOdkv, batch 4, keep-alive "
                    f"2 s; sources in pinned host memory; pools on {'devices 0..3' if ngpu >= 4 else 'this one GPU'}",
        "modes": modes,
        "note": "run_s = wall time of Simulator::run (every pool's data plane included: async loads complete "
                "before the pools report); peer mode uses the peer-aware schedule (estimate (S-S'-S'_peer)/B_pcie + "
                "S'_peer/B_nvlink, B_nvlink = 700 GB/s) and TG_LOAD_PEER — its RunMetrics differ from the "
                "reference's by design"}
    return out


def check_parity(tg, pool, target, host, cache, dev):
    """Decisions/dump vs the compiled reference (if present) and placed bytes
    vs the CPU restatement of tgfp1."""
    out = {}
    from oracle import cpu
    info = {t.id: pool.tensor_info(t.id) for t in target.tensors}
    ok = True
    for tid, pb in host.items():
        want, _ = cpu.content_fingerprint(pb.ptr, 16, n=pb.n)
        ok &= info[tid]["digest"] == want
    out["placed_digests_match_cpu_oracle"] = bool(ok)
    try:
        from oracle import ref
        if ref.available():
            rcat = {m["model_id"]: m for m in ref.default_catalog()}
            st = ref.ReuseStore(POOL, gpu_id=f"gpu{dev}")
            stats = ref.ModelStatsTable()
            for i, mid in enumerate(SEQ):
                stats.record_request(mid, 10.0 * i)
                stats.set_load_bandwidth(mid, 55e9)
                st.load_model(rcat[mid], stats, 10.0 * i)
                if i < 2:
                    st.end_instance(mid)
            out["dump_equals_reference"] = st.dump() == pool.dump()
    except Exception as e:  # pragma: no cover
        out["dump_equals_reference"] = f"unavailable: {e}"
    return out


def cpu_baseline(args):
    from oracle import cpu, ref
    if not ref.available():
        return None
    threads = args.cpu_threads or os.cpu_count()
    rcat, arena, sources, keep = cpu_setup(ref, cpu, threads)
    cpu_load_once(ref, cpu, rcat, arena, sources, threads)
    times = [cpu_load_once(ref, cpu, rcat, arena, sources, threads)[0] for _ in range(5)]
    sec = statistics.median(times)
    total = rcat[SEQ[2]]["total_size"]
    return {"value": total / sec / 1e9, "unit": "GB/s", "cores": threads, "kind": "port",
            "ms_per_step": sec * 1e3, "ms_all": [t * 1e3 for t in times], "host_ram_gib": host_ram_gib(),
            "sample": f"median of 5 timed replays of load #3 (after 1 untimed) on a {POOL >> 30} GiB host arena: "
                      f"reference ReuseStore::load_model (oracle/_ref) + CPU data plane port (memmove relocations, "
                      f"memcpy placements, tgfp1 of all {len(rcat[SEQ[2]]['tensors'])} tensors), {threads} threads"}


def measure_p2p_peak(local, peer, n=1 << 30, reps=5):
    """The NVLink roofline of the peer pull, measured in this run: a plain
    copy-engine copy (torch, cudaMemcpyPeerAsync underneath) of n bytes from
    the neighbour GPU's memory into this GPU's, best of `reps`, CUDA events on
    the local stream.  Every rank runs it at the same time, reading its right
    neighbour — the peer pull's own traffic pattern.  On a shared-GPU flow
    check the "peer" is this device (a D2D copy, labelled as such)."""
    import torch
    src = torch.empty(n, dtype=torch.uint8, device=f"cuda:{peer}")
    dst = torch.empty(n, dtype=torch.uint8, device=f"cuda:{local}")
    s = torch.cuda.current_stream(local)
    best = 1e9
    for r in range(reps + 1):
        torch.cuda.synchronize(local)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        dst.copy_(src, non_blocking=True)
        b.record(s)
        b.synchronize()
        if r:
            best = min(best, a.elapsed_time(b))
    del src, dst
    torch.cuda.empty_cache()
    return n / (best / 1e3) / 1e9


def c4_measure(tg, rank, world, local, steps, warmup):
    """C4: GPT-20B tensor-sharded over N ranks.  Cold: every rank
    loads its shard (40e9/N bytes) from pinned host memory over its own PCIe
    link, no collective.  Peer (N > 1): ranks exchange CUDA IPC arena handles
    and indexes (all_gather_object), then each rank loads its right
    neighbour's shard — every byte is pulled from the neighbour's pool over
    NVLink by the load kernel and fingerprint-verified against the
    neighbour's digest.  The NVLink roofline is a copy-engine peer copy
    measured in the same run.  Collective calls match on every rank; returns
    the max-over-ranks result (all ranks)."""
    import torch.distributed as dist
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    gpt = catalog(tg)["gpt20B"]
    mine = tg.shard_model(gpt, rank, world)
    right = tg.shard_model(gpt, (rank + 1) % world, world)
    peer_dev = local if shared_gpu() else (local + 1) % world  # one node: device = local rank
    p2p_peak = None
    if world > 1:
        dist.barrier()
        p2p_peak = measure_p2p_peak(local, peer_dev)
    h2d_peak = measured_h2d_peak(local)
    pool = tg.ReuseStore(tg.GpuSpec(f"gpu{local}", mine.total_size + right.total_size + GIB), device=local)
    cold_ms, peer_ms, peer_bytes, verify, kernel_ms = [], [], 0, 0, []
    with HostCheckpoint([mine], device=local):
        for step in range(warmup + steps):
            pool.evict_model(right.model_id)
            pool.end_instance(mine.model_id)
            pool.evict_model(mine.model_id)
            st = tg.ModelStatsTable()
            st.record_request(mine.model_id, 0.0)
            if world > 1:
                dist.barrier()
            ms, o = _event_ms(pool.stream(), local, lambda: pool.load_model(mine, st, 0.0, details=False).value())
            if step >= warmup:
                cold_ms.append(ms)
            verify += o.verify_mismatches
            if world > 1:
                peers = [None] * world
                dist.all_gather_object(peers, (pool.export_ipc(), pool.index()))
                if step == 0:
                    pid = {r: pool.attach_remote(*peers[r]) for r in range(world) if r != rank}
                else:
                    for r, p in pid.items():
                        pool.update_remote(p, peers[r][1])
                st.record_request(right.model_id, 1.0)
                dist.barrier()
                ms, o = _event_ms(pool.stream(), local, lambda: pool.load_model(
                    right, st, 1.0, tg.LoadPolicy(flags=1 | 2 | 4 | 8), details=False).value())
                if step >= warmup:
                    peer_ms.append(ms)
                    kernel_ms.append(o.timings["relocate_ms"])
                peer_bytes = o.peer_bytes
                verify += o.verify_mismatches
                dist.barrier()
    mc = statistics.mean(cold_ms)
    mp_ = statistics.mean(peer_ms) if peer_ms else None
    mk = statistics.mean(kernel_ms) if kernel_ms else None
    per_rank_verify = [verify]
    if world > 1:
        per_rank_verify = [None] * world
        dist.all_gather_object(per_rank_verify, verify)
        mc, mp_, mk = reduce_max([mc, mp_ or 0.0, mk or 0.0], local)
        p2p_peak = reduce_max([-p2p_peak], local)[0] * -1  # the slowest rank's link
        h2d_peak = reduce_max([-h2d_peak], local)[0] * -1
    pool.close()
    peer = None
    if mp_:
        ach = peer_bytes / (mp_ / 1e3) / 1e9
        peer = {"what": "each rank loads its right neighbour's shard from the neighbour's pool (CUDA IPC + the load "
                        "kernel over NVLink), every byte fingerprint-verified against the neighbour's digest",
                "bytes_per_rank": peer_bytes, "ms": mp_, "load_kernel_ms": mk,
                "per_rank_GBps": ach, "aggregate_GBps": world * ach,
                "roofline": {"bound": "nvlink", "achieved": ach, "peak": p2p_peak, "unit": "GB/s",
                             "frac": ach / p2p_peak if p2p_peak else None,
                             "peak_source": ("D2D copy on the shared GPU (flow check, not NVLink)" if shared_gpu()
                                             else "copy-engine peer copy of 1 GiB from the right neighbour, all ranks "
                                                  "at once, measured in this run (min over ranks)")}}
    return {"workload": "C4 GPT-20B sharded 1/N per rank (shard r = bytes [r*ceil(n/N), ...) of every tensor)",
            "n_ranks": world, "steps": steps, "warmup": warmup, "shard_bytes_rank0": mine.total_size,
            "cold_ms": mc, "cold_aggregate_GBps": gpt.total_size / (mc / 1e3) / 1e9,
            "cold_per_rank_GBps": mine.total_size / (mc / 1e3) / 1e9,
            "cold_roofline": {"bound": "pcie", "achieved": mine.total_size / (mc / 1e3) / 1e9, "peak": h2d_peak,
                              "unit": "GB/s", "frac": mine.total_size / (mc / 1e3) / 1e9 / h2d_peak,
                              "peak_source": "pinned H2D 2 GiB per rank in this run (min over ranks)"},
            "peer": peer, "verify_mismatches_per_rank": per_rank_verify}


def run_c4(args):
    """--workload c4: the C4 measurement as the bench line."""
    import torch.distributed as dist
    rank, world, local = dist_setup()
    import paper_2512_01357_b200 as tg
    r = c4_measure(tg, rank, world, local, args.steps, args.warmup)
    if rank == 0:
        gpt = catalog(tg)["gpt20B"]
        line = {"metric": "GPT-20B tensor-sharded cold load, aggregate GB/s (40e9 B over N PCIe links)",
                "value": r["cold_aggregate_GBps"], "unit": "GB/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["cold_ms"], "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
                "config": {"workload": r["workload"], "shard_bytes_rank0": r["shard_bytes_rank0"],
                           "model_bytes": gpt.total_size, "parallelism": f"tp{world} shards, independent pools"},
                "peer": r["peer"], "verify_mismatches": r["verify_mismatches"]}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_launch(args):
    """`--gpus N` without torchrun: launch the N ranks ourselves (one process
    per GPU, the same command line) and pass rank 0's line through."""
    if not shared_gpu():
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible "
                             f"(TANGRAM_BENCH_SHARED_GPU=1 runs the N-rank flow on one GPU)")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    global POOL, SEQ
    args = parse()
    world_env = os.environ.get("WORLD_SIZE")
    if args.impl == "reference" and world_env is None:
        return run_reference_arm(args)  # the CPU path: one process, no ranks to launch
    if world_env is None and args.gpus > 1:
        return self_launch(args)
    if world_env is not None and int(world_env) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}: launch one rank per GPU")
    if shared_gpu():  # flow check of N > 1 on one GPU: a switch small enough for N copies
        POOL, SEQ = 7 * GIB, ["qwen3B", "opt1.3B", "qwen3B"]  # 9 relocations, 1.2 GB placed
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.workload == "c4":
        return run_c4(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
