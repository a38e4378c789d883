"""C4 at full size on a device (SURVEY §8(d) C4, §8(e) parity row): the
GPT-20B tensor-parallel shard of one rank (TP2: 20 GB) loaded cold into a
160 GiB device pool from pinned host memory, then reloaded at 100 % reuse.

* Decisions: the dump equals the compiled reference's ReuseStore run on the
  same shard ModelSpec (reuse_store.hpp:120-174).
* Bytes: every shard tensor's device tgfp1 (from the load and re-measured on
  the resident bytes) equals the CPU restatement of its byte range of the
  parent tensor, generated on the CPU independently of the device synth.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

POOL = 160 << 30


def _cpu_shard_digest(cpu, tg, t, scratch):
    parent, begin, size = tg.lineage(t.id)
    assert size == t.size
    buf = scratch[:size]
    cpu.synth_into(parent.hi, parent.lo, buf.ctypes.data, size, begin)
    return cpu.content_fingerprint(buf, threads=16)[0]


@pytest.mark.parametrize("rank", [0, 1])
def test_c4_gpt20b_tp2_shard_on_device(tg, cpu, ref, rank):
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    cat = {m.model_id: m for m in tg.default_catalog()}
    shard = tg.shard_model(cat["gpt20B"], rank, 2)
    assert len(shard.tensors) == 45 and abs(shard.total_size - 20_000_000_000) < 64
    scratch = np.empty(max(t.size for t in shard.tensors), dtype=np.uint8)
    want = [_cpu_shard_digest(cpu, tg, t, scratch) for t in shard.tensors]
    pool = tg.ReuseStore(tg.GpuSpec(f"gpu{rank}", POOL), device=0)
    st = tg.ModelStatsTable()
    r_pool, r_st = ref.ReuseStore(POOL, gpu_id=f"gpu{rank}"), ref.ModelStatsTable()
    try:
        with HostCheckpoint([shard]):
            st.record_request(shard.model_id, 0.0)
            cold = pool.load_model(shard, st, 0.0).value()
            assert cold.pcie_bytes == shard.total_size and cold.bytes_transferred == shard.total_size
            assert cold.digests == want
            r_st.record_request(shard.model_id, 0.0)
            r_pool.load_model(shard.to_json(), r_st, 0.0)
            assert pool.dump() == r_pool.dump()
            pool.end_instance(shard.model_id)
            r_pool.end_instance(shard.model_id)
            st.record_request(shard.model_id, 1.0)
            warm = pool.load_model(shard, st, 1.0).value()
            assert warm.bytes_transferred == 0 and warm.verify_mismatches == 0
            assert warm.fingerprint_bytes == shard.total_size and warm.digests == want
            r_st.record_request(shard.model_id, 1.0)
            r_pool.load_model(shard.to_json(), r_st, 1.0)
            assert pool.dump() == r_pool.dump()
        for i, t in enumerate(shard.tensors):
            assert pool.fingerprint_tensor(t.id) == want[i], t.name
        print(f"rank {rank}: cold {cold.timings['total_ms']:.1f} ms "
              f"({shard.total_size / cold.timings['total_ms'] / 1e6:.1f} GB/s), "
              f"warm {warm.timings['total_ms']:.2f} ms")
    finally:
        pool.close()
