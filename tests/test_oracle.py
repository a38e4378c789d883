"""Pin the oracle before trusting it.

* oracle/_ref (the reference compiled from /root/reference) must reproduce
  the known-answer vectors of SURVEY Appendix A / SPEC examples (committed in
  tests/golden/known_answers.json);
* oracle/cpu_oracle.c (the plain-C restatement) must agree with the compiled
  reference's murmur3 on random inputs and with the canonical MurmurHash3
  vector, and the tgfp1 fingerprint must be invariant to threading.
"""
import json
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _kat():
    with open(os.path.join(GOLDEN, "known_answers.json")) as f:
        return json.load(f)


def test_cpu_murmur3_canonical_vector(cpu):
    h = cpu.murmur3(b"hello")
    assert "%016x%016x" % h == "cbd8a7b341bd9b025b1e906a48ae1d19"
    assert cpu.murmur3(b"") == (0, 0)


def test_cpu_murmur3_matches_reference(cpu, ref):
    rng = np.random.default_rng(3)
    for n in list(range(0, 70)) + [255, 256, 4095, 4096, 4097, 10000]:
        d = rng.integers(0, 256, size=n, dtype=np.uint8).tobytes()
        for seed in (0, 1, 12345, 2**63 + 7):
            assert cpu.murmur3(d, seed) == ref.murmur3(d, seed)


def test_reference_known_answers(ref):
    kat = _kat()
    assert "%016x%016x" % ref.murmur3(b"hello") == kat["murmur3_hello"]
    assert ref.fingerprint("opt1.3B", "layer0.qkv", [2048, 6144]) == kat["fingerprint_opt13_layer0_qkv"]
    cat = {m["model_id"]: m for m in ref.default_catalog()}
    cat["llama2-13B"] = ref.make_model("llama2-13B", 26_000_000_000, 40, 819_200)
    # Appendix A table, independent of the generated fixture
    appendix_a = {
        "opt1.3B": [2_600_000_000, 25, 68_611_111, 137_222_226, 26_624],
        "qwen3B": [6_000_000_000, 27, 146_153_846, 300_000_000, 60_416],
        "llama3B": [6_000_000_000, 27, 146_153_846, 300_000_000, 60_416],
        "opt6.7B": [13_400_000_000, 33, 265_208_333, 670_000_000, 134_144],
        "llama8B": [16_000_000_000, 33, 316_666_666, 800_000_000, 160_768],
        "yi9B": [18_000_000_000, 37, 316_666_666, 900_000_000, 180_224],
        "opt13B": [26_000_000_000, 41, 411_666_666, 1_300_000_000, 260_096],
        "gpt20B": [40_000_000_000, 45, 575_757_575, 2_000_000_000, 400_384],
        "llama2-13B": [26_000_000_000, 81, 205_833_333, 1_300_000_000, 819_200],
    }
    assert kat["catalog"] == appendix_a
    assert kat["murmur3_hello"] == "cbd8a7b341bd9b025b1e906a48ae1d19"
    assert kat["fingerprint_opt13_layer0_qkv"] == "67a2b7bfa70bad4d53297840b8fe3b41"
    assert kat["opt13_first_tensor_id"] == "4396475c6c12402a507c13a93d0841f1"
    for mid, row in kat["catalog"].items():
        m = cat[mid]
        sizes = [t["size"] for t in m["tensors"]]
        assert [m["total_size"], len(m["tensors"]), min(sizes), max(sizes), m["bytes_per_token"]] == row
    assert cat["opt1.3B"]["tensors"][0]["id"] == kat["opt13_first_tensor_id"]


def test_content_fingerprint_thread_invariant(cpu):
    rng = np.random.default_rng(5)
    for n in (0, 1, 4096, 4097, 1 << 20, (1 << 20) + 333):
        d = rng.integers(0, 256, size=n, dtype=np.uint8)
        a = cpu.content_fingerprint(d, threads=1)
        b = cpu.content_fingerprint(d, threads=7)
        assert a == b


def test_content_fingerprint_definition(cpu):
    """tgfp1 spelled out in Python over the oracle's murmur3 (small case)."""
    rng = np.random.default_rng(9)
    d = rng.integers(0, 256, size=3 * 4096 + 100, dtype=np.uint8)
    H = L = 0
    for i in range(4):
        leaf = d[i * 4096:(i + 1) * 4096].tobytes()
        h, l = cpu.murmur3(leaf, i)
        H, L = (H + h) % 2**64, (L + l) % 2**64
    root = cpu.murmur3(H.to_bytes(8, "little") + L.to_bytes(8, "little") + d.size.to_bytes(8, "little"), 0)
    assert cpu.content_fingerprint(d)[0] == root
    assert cpu.content_fingerprint(d)[1] == (H, L)


def test_synth_stream_definition(cpu):
    tid = (0x0123456789ABCDEF, 0xFEDCBA9876543210)
    seed = tid[0] ^ (((tid[1] << 17) | (tid[1] >> 47)) & (2**64 - 1))

    def splitmix(z):
        z = (z + 0x9E3779B97F4A7C15) % 2**64
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) % 2**64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) % 2**64
        return z ^ (z >> 31)

    want = b"".join(splitmix(seed ^ ((w * 0x9E3779B97F4A7C15) % 2**64)).to_bytes(8, "little") for w in range(8))
    assert cpu.synth(*tid, 64).tobytes() == want
    assert cpu.synth(*tid, 13, begin=5).tobytes() == want[5:18]
