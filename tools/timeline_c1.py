"""Kernel / memcpy timeline of C1 loads (OPT-1.3B cold from pinned host, then
the 100 % reuse reload), from CUPTI via torch.profiler, untimed diagnostics.
Prints one JSON object: per load the device events with start / duration
relative to the first one, and the CUDA-event latency of the load.

    python tools/timeline_c1.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile
    import paper_2512_01357_b200 as tg
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    dev = 0
    m = {x.model_id: x for x in tg.default_catalog()}["opt1.3B"]
    pool = tg.ReuseStore(tg.GpuSpec("gpu0", 8 << 30), device=dev)
    stream = torch.cuda.ExternalStream(pool.stream(), device=dev)
    out = {}
    with HostCheckpoint([m], device=dev):
        stats = tg.ModelStatsTable()
        t = 0.0
        for rnd in range(2):
            for kind in ("cold", "warm"):
                if kind == "cold":
                    pool.evict_model(m.model_id)
                stats.record_request(m.model_id, t)
                torch.cuda.synchronize()
                with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    o = pool.load_model(m, stats, t, details=False).value()
                    b.record(stream)
                    b.synchronize()
                pool.end_instance(m.model_id)
                t += 1.0
                if rnd == 0:
                    continue
                evs = []
                for e in prof.events():
                    if e.device_type.name != "CUDA":
                        continue
                    evs.append({"name": e.name[:60], "start_us": e.time_range.start,
                                "dur_us": round(e.time_range.elapsed_us(), 2)})
                t0 = min((e["start_us"] for e in evs), default=0)
                for e in evs:
                    e["start_us"] = round(e["start_us"] - t0, 2)
                evs.sort(key=lambda e: e["start_us"])
                out[kind] = {"event_ms": a.elapsed_time(b), "timings": o.timings, "device_events": evs}
    pool.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
