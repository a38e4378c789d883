"""Generate the golden fixtures of tests/golden from the REFERENCE itself.

Run here (where /root/reference exists): builds nothing, uses oracle/_ref
(the unmodified reference headers compiled by oracle/Makefile).  Fixtures:
  known_answers.json  — SURVEY Appendix A / SPEC known answers, re-derived
  c1_c2_loads.json    — per-load LoadOutcome + final dump for C1/C2 sweeps
  c3_kv.json          — KV burst tables / address tables for C3 (16, 64 req)
  c5_sim.json         — reference Simulator aggregates for the C5 config
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import ref  # noqa: E402

GIB = 1 << 30


def dump(name, obj):
    with open(os.path.join(HERE, name), "w") as f:
        json.dump(obj, f, separators=(",", ":"), sort_keys=True)
        f.write("\n")


def known_answers():
    cat = ref.default_catalog()
    rows = {}
    for m in cat:
        s = [t["size"] for t in m["tensors"]]
        rows[m["model_id"]] = [m["total_size"], len(m["tensors"]), min(s), max(s), m["bytes_per_token"]]
    l2 = ref.make_model("llama2-13B", 26_000_000_000, 40, 819_200)
    s = [t["size"] for t in l2["tensors"]]
    rows["llama2-13B"] = [l2["total_size"], len(l2["tensors"]), min(s), max(s), l2["bytes_per_token"]]
    return {
        "murmur3_hello": "%016x%016x" % ref.murmur3(b"hello"),
        "fingerprint_opt13_layer0_qkv": ref.fingerprint("opt1.3B", "layer0.qkv", [2048, 6144]),
        "catalog": rows,
        "opt13_first_tensor_id": cat[0]["tensors"][0]["id"],
        "catalog_ids": {m["model_id"]: [t["id"] for t in m["tensors"]] for m in cat},
    }


def switch_sequence(pool_bytes, seq, merge=0, strictness=0):
    cat = {m["model_id"]: m for m in ref.default_catalog()}
    st = ref.ReuseStore(pool_bytes)
    stats = ref.ModelStatsTable()
    out = []
    t = 0.0
    for mid in seq:
        stats.record_request(mid, t)
        stats.set_load_bandwidth(mid, 55e9)
        o = st.load_model(cat[mid], stats, t, merge=merge, strictness=strictness)
        out.append(o)
        st.end_instance(mid)
        t += 10.0
    return {"loads": out, "final_dump": st.dump()}


def c3_kv(n_requests_list=(16, 64)):
    res = {}
    model = ref.make_model("llama2-13B", 26_000_000_000, 40, 819_200)
    for n in n_requests_list:
        st = ref.ReuseStore(160 * GIB)
        stats = ref.ModelStatsTable()
        stats.record_request("llama2-13B", 0.0)
        st.load_model(model, stats, 0.0)
        kv = ref.KvEngine("llama2-13B", 16, 819_200)
        prompts = [min(p, 8192) for p, _ in ref.sample_lengths(7, "sharegpt", n)]
        reqs = [(i + 1, p) for i, p in enumerate(prompts)]
        burst = kv.batch_allocate(st, stats, reqs)
        decode = kv.batch_allocate(st, stats, [(i + 1, (p + 15) // 16 * 16 + 1) for i, p in enumerate(prompts)])
        tables = {str(i + 1): kv.table(i + 1) for i in range(n)}
        res[str(n)] = {"requests": reqs, "burst": burst["granted"], "decode": decode["granted"],
                       "state": kv.state(), "tables": tables, "info": st.info(),
                       "regions": len(st.dump()["regions"])}
    return res


def main():
    dump("known_answers.json", known_answers())
    seq = ["opt13B", "opt6.7B", "opt13B", "opt6.7B", "opt13B"]
    loads = {}
    for gib in (30, 32, 36, 40):
        loads[f"pg_{gib}"] = switch_sequence(gib * GIB, seq)
    for gib in (32, 36):
        loads[f"gm_{gib}"] = switch_sequence(gib * GIB, seq, merge=1)
    loads["lg_32"] = switch_sequence(32 * GIB, seq, strictness=1)
    c1 = switch_sequence(160 * GIB, ["opt1.3B", "opt1.3B"])
    loads["c1_160"] = c1
    dump("c1_c2_loads.json", loads)
    dump("c3_kv.json", c3_kv())
    sim = {}
    for mode in ("baseline", "reuse", "reuse_odkv"):
        r = ref.simulate({"trace": {"seed": 42, "num_requests": 2000, "locality": "L3", "mean_interarrival": 0.5,
                                    "zipf_s": 1.1, "repeat_probability": 0.6},
                          "sim": {"n_gpus": 8, "pool_size": 48 * GIB, "mode": mode, "batch_size": 4,
                                  "keep_alive": 2.0}})
        r.pop("ns")
        sim[mode] = r
    dump("c5_sim.json", sim)


if __name__ == "__main__":
    main()
