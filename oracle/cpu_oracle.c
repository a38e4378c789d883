/* ORACLE / TEST INFRASTRUCTURE ONLY — the checker, never the product.
 *
 * Plain-C CPU restatement of the byte-level parts of the Tangram load path
 * that the reference (/root/reference/proj/include/warmsim) does not execute
 * because it moves no bytes.  Built by oracle/Makefile into
 * oracle/_build/libtangram_oracle.so and loaded only by tests/, by
 * __graft_entry__.smoke() (as the checker) and by bench.py's cpu_baseline /
 * --impl reference leg.
 *
 *  - orc_murmur3_x64_128: MurmurHash3 x64-128, restated from
 *      types.hpp:64-124 (rotl64 64, fmix64 66-73, body 86-95, tail 97-117,
 *      finalisation 119-123).  Pinned against the reference itself through
 *      oracle/_ref (tests/test_oracle.py) and the canonical published vector
 *      murmur3("hello", seed 0) = cbd8a7b341bd9b025b1e906a48ae1d19.
 *  - orc_content_fingerprint: the content fingerprint "tgfp1" (SURVEY §8 a2′,
 *      no reference counterpart): leaf_i = murmur3(bytes[4096 i, 4096 i+4096)
 *      ∩ [0,n), seed=i); (H,L) = (Σ leaf.hi, Σ leaf.lo) mod 2^64;
 *      root = murmur3(le64 H ‖ le64 L ‖ le64 n, seed=0).
 *  - orc_synth_fill: the synthetic checkpoint byte stream:
 *      little-endian u64 word w of tensor t is
 *      splitmix64(t.hi ^ rotl(t.lo,17) ^ (w * 0x9E3779B97F4A7C15)).
 *  - orc_replay_*: the CPU data plane of ReuseStore::apply_plan
 *      (reuse_store.hpp:316-334): relocations as copies in plan order,
 *      placements as copies from the host checkpoint, multithreaded.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_LEAF 4096u

static inline uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

static inline uint64_t fmix64(uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdULL;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ULL;
    k ^= k >> 33;
    return k;
}

void orc_murmur3_x64_128(const void *key, uint64_t len, uint64_t seed, uint64_t out[2]) {
    const uint8_t *data = (const uint8_t *)key;
    const uint64_t nblocks = len / 16;
    uint64_t h1 = seed, h2 = seed;
    const uint64_t c1 = 0x87c37b91114253d5ULL, c2 = 0x4cf5ad432745937fULL;
    for (uint64_t i = 0; i < nblocks; i++) {
        uint64_t k1, k2;
        memcpy(&k1, data + i * 16, 8);
        memcpy(&k2, data + i * 16 + 8, 8);
        k1 *= c1; k1 = rotl64(k1, 31); k1 *= c2; h1 ^= k1;
        h1 = rotl64(h1, 27); h1 += h2; h1 = h1 * 5 + 0x52dce729;
        k2 *= c2; k2 = rotl64(k2, 33); k2 *= c1; h2 ^= k2;
        h2 = rotl64(h2, 31); h2 += h1; h2 = h2 * 5 + 0x38495ab5;
    }
    const uint8_t *tail = data + nblocks * 16;
    const unsigned rem = (unsigned)(len & 15);
    uint64_t k1 = 0, k2 = 0;
    /* Same accumulation as the reference's fallthrough switch. */
    for (unsigned b = rem; b > 8; --b) k2 ^= (uint64_t)tail[b - 1] << (8 * (b - 9));
    if (rem > 8) { k2 *= c2; k2 = rotl64(k2, 33); k2 *= c1; h2 ^= k2; }
    for (unsigned b = rem < 8 ? rem : 8; b > 0; --b) k1 ^= (uint64_t)tail[b - 1] << (8 * (b - 1));
    if (rem > 0) { k1 *= c1; k1 = rotl64(k1, 31); k1 *= c2; h1 ^= k1; }
    h1 ^= len; h2 ^= len;
    h1 += h2; h2 += h1;
    h1 = fmix64(h1); h2 = fmix64(h2);
    h1 += h2; h2 += h1;
    out[0] = h1;
    out[1] = h2;
}

/* Leaf sums over leaves [l0, l1) of a tensor of n bytes. */
static void leaf_sums(const uint8_t *p, uint64_t n, uint64_t l0, uint64_t l1, uint64_t *H, uint64_t *L) {
    uint64_t h = 0, l = 0;
    for (uint64_t i = l0; i < l1; ++i) {
        const uint64_t off = i * ORC_LEAF;
        const uint64_t len = (n - off) < ORC_LEAF ? (n - off) : ORC_LEAF;
        uint64_t d[2];
        orc_murmur3_x64_128(p + off, len, i, d);
        h += d[0];
        l += d[1];
    }
    *H = h;
    *L = l;
}

void orc_fingerprint_finalize(uint64_t H, uint64_t L, uint64_t n, uint64_t out[2]) {
    uint8_t buf[24];
    memcpy(buf, &H, 8); /* little-endian host (x86-64) */
    memcpy(buf + 8, &L, 8);
    memcpy(buf + 16, &n, 8);
    orc_murmur3_x64_128(buf, 24, 0, out);
}

typedef struct {
    const uint8_t *p;
    uint64_t n, l0, l1, H, L;
} fp_job;

static void *fp_worker(void *arg) {
    fp_job *j = (fp_job *)arg;
    leaf_sums(j->p, j->n, j->l0, j->l1, &j->H, &j->L);
    return NULL;
}

/* Content fingerprint of n bytes at p using up to `threads` host threads.
 * Also returns the leaf sums (H, L) when sums != NULL. */
void orc_content_fingerprint(const void *p, uint64_t n, int threads, uint64_t out[2], uint64_t sums[2]) {
    const uint64_t leaves = (n + ORC_LEAF - 1) / ORC_LEAF;
    if (threads < 1) threads = 1;
    if ((uint64_t)threads > leaves) threads = leaves ? (int)leaves : 1;
    uint64_t H = 0, L = 0;
    if (threads == 1) {
        leaf_sums((const uint8_t *)p, n, 0, leaves, &H, &L);
    } else {
        pthread_t tid[256];
        fp_job jobs[256];
        if (threads > 256) threads = 256;
        for (int t = 0; t < threads; ++t) {
            jobs[t].p = (const uint8_t *)p;
            jobs[t].n = n;
            jobs[t].l0 = leaves * t / threads;
            jobs[t].l1 = leaves * (t + 1) / threads;
            pthread_create(&tid[t], NULL, fp_worker, &jobs[t]);
        }
        for (int t = 0; t < threads; ++t) {
            pthread_join(tid[t], NULL);
            H += jobs[t].H;
            L += jobs[t].L;
        }
    }
    if (sums) { sums[0] = H; sums[1] = L; }
    orc_fingerprint_finalize(H, L, n, out);
}

static inline uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* Bytes [begin, begin+len) of the synthetic tensor (hi, lo). */
void orc_synth_fill(uint64_t hi, uint64_t lo, uint64_t begin, uint64_t len, void *dst) {
    const uint64_t seed = hi ^ rotl64(lo, 17);
    uint8_t *out = (uint8_t *)dst;
    uint64_t pos = begin;
    const uint64_t end = begin + len;
    while (pos < end) {
        const uint64_t w = pos / 8;
        const uint64_t v = splitmix64(seed ^ (w * 0x9E3779B97F4A7C15ULL));
        const unsigned b0 = (unsigned)(pos % 8);
        unsigned nb = 8 - b0;
        if (nb > end - pos) nb = (unsigned)(end - pos);
        memcpy(out + (pos - begin), ((const uint8_t *)&v) + b0, nb);
        pos += nb;
    }
}

typedef struct {
    uint8_t *dst;
    const uint8_t *src;
    uint64_t len;
} cp_job;

static void *cp_worker(void *arg) {
    cp_job *j = (cp_job *)arg;
    memcpy(j->dst, j->src, j->len);
    return NULL;
}

/* Parallel copy of disjoint ranges (relocation source and destination are
 * disjoint by construction: RegionList::move rejects overlap,
 * region_pool.hpp:157-167). */
void orc_copy(void *dst, const void *src, uint64_t len, int threads) {
    if (threads <= 1 || len < (1u << 20)) {
        memmove(dst, src, len);
        return;
    }
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    cp_job jobs[256];
    for (int t = 0; t < threads; ++t) {
        const uint64_t a = len * t / threads, b = len * (t + 1) / threads;
        jobs[t].dst = (uint8_t *)dst + a;
        jobs[t].src = (const uint8_t *)src + a;
        jobs[t].len = b - a;
        pthread_create(&tid[t], NULL, cp_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
}

/* CPU replay of one plan's data movement on a host arena (reuse_store.hpp:
 * 323-333): relocations in plan order, then placements from host sources. */
void orc_replay_plan(uint8_t *arena, uint64_t n_reloc, const uint64_t *reloc /* from,to,size triples */,
                     uint64_t n_place, const uint64_t *place /* offset,size pairs */, const void *const *srcs,
                     int threads) {
    for (uint64_t i = 0; i < n_reloc; ++i)
        orc_copy(arena + reloc[3 * i + 1], arena + reloc[3 * i], reloc[3 * i + 2], threads);
    for (uint64_t i = 0; i < n_place; ++i) orc_copy(arena + place[2 * i], srcs[i], place[2 * i + 1], threads);
}
