"""The reuse sweep of bench.py alone (C2 load #3 at 30/32/36/40 GiB; value +
e2e, with the device timeline of the gated H2D):  -> gpurun_out/reuse_sweep.json"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
import paper_2512_01357_b200 as tg  # noqa: E402

peak = bench.measured_h2d_peak(0)
r = bench.run_reuse_sweep(tg, 0, peak)
r["h2d_peak_GBps"] = peak
os.makedirs("gpurun_out", exist_ok=True)
json.dump(r, open("gpurun_out/reuse_sweep.json", "w"), indent=1)
for k, v in r["pools"].items():
    print(k, round(v["reuse_ratio"], 4), {n: (round(v[n]["ms"], 3), v[n].get("frac_of_pcie_floor"), v[n]["timeline_ms"])
                                          for n in ("value", "e2e")})
