"""Turn raw ncu outputs from gpurun_out/ into the committed summaries under
profiles/ (the .ncu-rep files stay in gpurun_out/, which is scratch).

    python tools/make_profiles.py r01
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_summary import summarise  # noqa: E402


def load_kernel_stalls(rep):
    """Issue activity, DRAM rate and warp-stall shares of the load kernel's
    ncu --set full capture (PC-sampling counts normalised to 1)."""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    d = dict(zip(rows[0], rows[2]))
    units = dict(zip(rows[0], rows[1]))
    pre = "smsp__pcsamp_warps_issue_stalled_"
    st = {k[len(pre):]: float(v.replace(",", "")) for k, v in d.items()
          if k.startswith(pre) and not k.endswith("_not_issued") and v}
    tot = sum(st.values()) or 1.0
    num = lambda k: float(d[k].replace(",", ""))
    return {
        "kernel": d.get("Kernel Name"),
        "gpu__time_duration_ms": num("gpu__time_duration.sum") * {"ms": 1.0, "us": 1e-3, "ns": 1e-6}[units["gpu__time_duration.sum"]],
        "issue_active_pct": d.get("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
        "dram_throughput_pct": d.get("dram__throughput.avg.pct_of_peak_sustained_elapsed",
                                     d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")),
        "registers": d.get("launch__registers_per_thread"),
        "warps_active_pct": d.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "stall_share": dict(sorted(((k, round(v / tot, 3)) for k, v in st.items() if v / tot >= 0.005),
                                   key=lambda kv: -kv[1])),
    }


def launch_shares(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.DictReader(io.StringIO("".join(lines)))
    per = defaultdict(lambda: [0, 0.0])
    order = []
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("unnamed>::", "")
        ns = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ns = ns * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
        per[name][0] += 1
        per[name][1] += ns
        order.append((name, ns))
    total = sum(v[1] for v in per.values())
    return {"total_kernel_ms": total / 1e6, "launches": len(order),
            "by_kernel": {k: {"launches": v[0], "ms": v[1] / 1e6, "share": v[1] / total if total else 0}
                          for k, v in sorted(per.items(), key=lambda kv: -kv[1][1])}}


def _bytes(v):
    val, unit = v
    return float(val.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[unit]


def traffic(rep, out_path, algo=None, source=None):
    """DRAM traffic of the bench step's launches (load kernel + concurrent K1)
    against the step's algorithmic bytes (printed by the same bench --profile
    run)."""
    launches = summarise(rep)
    log = os.path.join(OUT, "prof_load.log")
    if algo is None and os.path.exists(log):
        for ln in open(log):
            if ln.startswith("{"):
                algo = json.loads(ln).get("roofline_step", {}).get("algorithmic_bytes_per_step")
    per = [{"ms": float(r["gpu__time_duration.sum"][0]) / (1e3 if r["gpu__time_duration.sum"][1] == "usecond" else 1),
            "dram_read_bytes": _bytes(r["dram__bytes_read.sum"]),
            "dram_write_bytes": _bytes(r["dram__bytes_write.sum"]),
            "dram_pct_of_peak": r["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"][0]} for r in launches]
    t = sum(x["dram_read_bytes"] + x["dram_write_bytes"] for x in per)
    with open(out_path, "w") as f:
        json.dump({"traffic_bytes_per_launch": t, "algorithmic_bytes": algo,
                   "ratio": t / algo if algo else None,
                   "source": source or "ncu --set full --clock-control none of the bench step's launches (bench.py --profile "
                             "--steps 1 --warmup 0): the load kernel and, since the verification split, the "
                             "concurrent K1 launch verifying the untouched reused tensors (ncu serialises them); "
                             "dram__bytes_read.sum + dram__bytes_write.sum summed over both",
                   "per_launch": per}, f, indent=1)


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    out = {}
    for name in sorted(os.listdir(OUT)):
        p = os.path.join(OUT, name)
        if name.endswith(".ncu-rep"):
            out[name] = summarise(p)
    if out:
        with open(os.path.join(PROF, f"{tag}_ncu_full.json"), "w") as f:
            json.dump(out, f, indent=1)
    lp = os.path.join(OUT, "launches.csv")
    if os.path.exists(lp):
        with open(os.path.join(PROF, f"{tag}_launches_summary.json"), "w") as f:
            json.dump(launch_shares(lp), f, indent=1)
        subprocess.run(["cp", lp, os.path.join(PROF, f"{tag}_launches.csv")])
    lk = os.path.join(OUT, "prof_load.ncu-rep")
    if os.path.exists(lk):
        traffic(lk, os.path.join(PROF, "load_kernel_traffic.json"))
        with open(os.path.join(PROF, f"{tag}_load_kernel_stalls.json"), "w") as f:
            json.dump(load_kernel_stalls(lk), f, indent=1)
    k3 = os.path.join(OUT, "prof_k3.ncu-rep")
    if os.path.exists(k3):
        traffic(k3, os.path.join(PROF, f"{tag}_k3_traffic.json"), algo=2 * (4 << 30),
                source="ncu --set full --clock-control none of K3 relocate_bulk_kernel moving 4 GiB src+0 -> dst+5 "
                       "(tools/kernel_bench.py --only reloc --gib 8); algorithmic = 4 GiB read + 4 GiB written")
        with open(os.path.join(PROF, f"{tag}_k3_stalls.json"), "w") as f:
            json.dump(load_kernel_stalls(k3), f, indent=1)
    for extra in ("kernel_bench.json", "bench.json"):
        p = os.path.join(OUT, extra)
        if os.path.exists(p):
            subprocess.run(["cp", p, os.path.join(PROF, f"{tag}_{extra}")])
    print(json.dumps(sorted(os.listdir(PROF))))


if __name__ == "__main__":
    main()
