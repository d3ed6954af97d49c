/* oracle/gx_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's hot path (Ginex "gx", header-only
 * C++20 under /root/reference/proj/include/gx). It is the CHECKER for the CUDA
 * path: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * may load it. The product (paper_2208_09151_b200/) never links or calls it.
 *
 * Parity of this restatement is pinned two ways (see tests/test_oracle.py):
 *   1. against the reference itself, compiled from its own headers into
 *      oracle/_ref/libgx_ref.so (oracle/Makefile, oracle/ref_driver.cpp);
 *   2. against committed golden fixtures in tests/golden/ generated from that
 *      same reference build (tests/golden/make_golden.py), plus the reference
 *      unit-test KATs restated in tests/test_kats.py.
 *
 * Every function cites the reference file:line it restates. Status codes
 * follow include/gx_b200.h (gx_status).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GXO_OK 0
#define GXO_INVALID_ARGUMENT 1
#define GXO_OUT_OF_RANGE 2
#define GXO_LOGIC_ERROR 3
#define GXO_RUNTIME_ERROR 4

#define PAGE 4096ULL
#define ITER_FLAG (1ULL << 63)
#define ITER_MASK (ITER_FLAG - 1)
#define ITER_DUMMY (~0ULL)

/* ---- RNG: common.hpp:68-101 ------------------------------------------- */
uint64_t gxo_mix64(uint64_t z) { /* common.hpp:90-95 */
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
uint64_t gxo_derive_seed(uint64_t base, uint64_t index) { /* common.hpp:99-101 */
    return gxo_mix64(base ^ gxo_mix64(index));
}
typedef struct { uint64_t s; } sm64;
static uint64_t sm_next(sm64* r) { /* common.hpp:72-77 */
    uint64_t z = (r->s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static uint64_t sm_bounded(sm64* r, uint64_t n) { /* common.hpp:80-83 */
    return (uint64_t)(((unsigned __int128)sm_next(r) * n) >> 64);
}

/* ---- page arithmetic: common.hpp:48-61 ---------------------------------- */
uint64_t gxo_pages_touched(uint64_t lo, uint64_t hi) {
    if (hi <= lo) return 0;
    return (hi - 1) / PAGE - lo / PAGE + 1;
}
uint64_t gxo_page_count_for_row(uint64_t row_bytes, uint64_t row) {
    uint64_t lo = row * row_bytes;
    return gxo_pages_touched(lo, lo + row_bytes);
}

/* ---- dataset synthesis: graphgen.hpp:32-77, graph_store.hpp:53-81 ------- */
/* generate_edges: floor(n*avg_degree) accepted RMAT edges; rejected attempts
 * still consume their `scale` draws (graphgen.hpp:55-70). */
int gxo_generate_edges(uint64_t n, double avg_deg, double a, double b, double c,
                       uint64_t seed, uint64_t* src, uint64_t* dst, uint64_t cap,
                       uint64_t* count) {
    if (n < 1 || avg_deg < 0) return GXO_INVALID_ARGUMENT;
    unsigned scale = 0;
    while ((1ULL << scale) < n) ++scale;
    uint64_t target = (uint64_t)(avg_deg * (double)n);
    *count = target;
    if (target > cap) return GXO_RUNTIME_ERROR;
    sm64 r = {seed};
    double ab = a + b, abc = a + b + c;
    uint64_t k = 0;
    while (k < target) {
        uint64_t s = 0, d = 0;
        for (unsigned lv = 0; lv < scale; ++lv) { /* rmat_edge, graphgen.hpp:32-50 */
            double x = (double)(sm_next(&r) >> 11) * 0x1.0p-53;
            s <<= 1;
            d <<= 1;
            if (x < a) {
            } else if (x < ab) {
                d |= 1;
            } else if (x < abc) {
                s |= 1;
            } else {
                s |= 1;
                d |= 1;
            }
        }
        if (s >= n || d >= n) continue;
        src[k] = s;
        dst[k] = d;
        ++k;
    }
    return GXO_OK;
}

static int cmp_u64(const void* x, const void* y) {
    uint64_t a = *(const uint64_t*)x, b = *(const uint64_t*)y;
    return a < b ? -1 : a > b;
}

/* build_csc (graph_store.hpp:53-81): per-destination sorted, deduplicated
 * in-neighbour lists. indices_out must hold m entries; *e = edges kept. */
int gxo_build_csc(uint64_t n, const uint64_t* src, const uint64_t* dst, uint64_t m,
                  uint64_t* indptr, uint64_t* indices_out, uint64_t* e) {
    for (uint64_t i = 0; i < m; ++i)
        if (src[i] >= n || dst[i] >= n) return GXO_OUT_OF_RANGE;
    uint64_t* cur = (uint64_t*)calloc(n + 1, 8);
    uint64_t* raw = (uint64_t*)malloc((m ? m : 1) * 8);
    for (uint64_t i = 0; i < m; ++i) cur[dst[i] + 1]++;
    for (uint64_t v = 0; v < n; ++v) cur[v + 1] += cur[v];
    uint64_t* nxt = (uint64_t*)malloc((n + 1) * 8);
    memcpy(nxt, cur, (n + 1) * 8);
    for (uint64_t i = 0; i < m; ++i) raw[nxt[dst[i]]++] = src[i];
    uint64_t k = 0;
    indptr[0] = 0;
    for (uint64_t v = 0; v < n; ++v) {
        uint64_t lo = cur[v], hi = cur[v + 1];
        qsort(raw + lo, hi - lo, 8, cmp_u64);
        for (uint64_t j = lo; j < hi; ++j)
            if (j == lo || raw[j] != raw[j - 1]) indices_out[k++] = raw[j];
        indptr[v + 1] = k;
    }
    *e = k;
    free(cur);
    free(raw);
    free(nxt);
    return GXO_OK;
}

float gxo_feature_value(uint64_t value_seed, uint64_t node, uint32_t col) { /* graphgen.hpp:74-77 */
    uint64_t h = gxo_mix64(value_seed ^ gxo_mix64(node * 0x10001ULL + col));
    return (float)(h >> 40) * 0x1.0p-24f;
}

/* ---- seed plans: sampler.hpp:48-65, pipeline.hpp:380-399 ---------------- */
int gxo_plan_seed_batches(const uint64_t* train, uint64_t n, uint64_t batch_size,
                          uint64_t epoch_seed, uint64_t* shuffled) {
    if (n == 0 || batch_size < 1) return GXO_INVALID_ARGUMENT;
    memcpy(shuffled, train, n * 8);
    sm64 r = {epoch_seed};
    for (uint64_t i = n - 1; i > 0; --i) {
        uint64_t j = sm_bounded(&r, i + 1);
        uint64_t t = shuffled[i];
        shuffled[i] = shuffled[j];
        shuffled[j] = t;
    }
    return GXO_OK;
}

/* derive_train_ids (pipeline.hpp:384-399); out must hold n entries scratch. */
uint64_t gxo_train_ids(uint64_t n, uint64_t seed, double frac, uint64_t* out) {
    uint64_t want = (uint64_t)((double)n * frac);
    if (want < 1) want = 1;
    if (want > n) want = n;
    for (uint64_t v = 0; v < n; ++v) out[v] = v;
    sm64 r = {gxo_derive_seed(gxo_mix64(seed) ^ 0x545241494EULL, 0)};
    for (uint64_t i = 0; i < want; ++i) {
        uint64_t j = i + sm_bounded(&r, n - i);
        uint64_t t = out[i];
        out[i] = out[j];
        out[j] = t;
    }
    qsort(out, want, 8, cmp_u64);
    return want;
}
uint64_t gxo_epoch_seed(uint64_t seed, uint64_t epoch) { /* pipeline.hpp:380-382 */
    return gxo_derive_seed(gxo_mix64(seed) ^ 0x45504F4348ULL, epoch);
}

/* ---- sampler: sampler.hpp:69-117 --------------------------------------- */
typedef struct {
    uint64_t* keys;
    uint32_t* vals;
    uint64_t cap, size;
} hmap;
#define HEMPTY (~0ULL)
static void hm_init(hmap* h, uint64_t cap) {
    h->cap = cap;
    h->size = 0;
    h->keys = (uint64_t*)malloc(cap * 8);
    h->vals = (uint32_t*)malloc(cap * 4);
    memset(h->keys, 0xff, cap * 8);
}
static uint64_t hm_slot(const hmap* h, uint64_t k) {
    uint64_t s = gxo_mix64(k) & (h->cap - 1);
    while (h->keys[s] != HEMPTY && h->keys[s] != k) s = (s + 1) & (h->cap - 1);
    return s;
}
static void hm_grow(hmap* h) {
    hmap n;
    hm_init(&n, h->cap * 2);
    for (uint64_t i = 0; i < h->cap; ++i)
        if (h->keys[i] != HEMPTY) {
            uint64_t s = hm_slot(&n, h->keys[i]);
            n.keys[s] = h->keys[i];
            n.vals[s] = h->vals[i];
            n.size++;
        }
    free(h->keys);
    free(h->vals);
    *h = n;
}
/* emplace: returns 1 if inserted; *val = mapped value either way. */
static int hm_emplace(hmap* h, uint64_t k, uint32_t v, uint32_t* val) {
    if (2 * (h->size + 1) > h->cap) hm_grow(h);
    uint64_t s = hm_slot(h, k);
    if (h->keys[s] == k) {
        *val = h->vals[s];
        return 0;
    }
    h->keys[s] = k;
    h->vals[s] = v;
    h->size++;
    *val = v;
    return 1;
}

/* sample_batch (sampler.hpp:69-117) over an in-memory CSC (indptr/indices as
 * the GraphFile would read them). IoStats charging follows
 * GraphFile::read_in_neighbors (graph_store.hpp:145-154): per expanded parent
 * one list, pages_touched(8*ip[v], 8*ip[v+1]), 8*deg bytes.
 * io[4] = {pages_read, rows_read, neighbor_lists_read, bytes_read}.
 * edges_out: (src_local, dst_local) u32 pairs, layers back to back. */
int gxo_sample_batch(const uint64_t* indptr, const uint64_t* indices, uint64_t n_nodes,
                     const uint64_t* seeds, uint64_t n_seeds, const uint32_t* fanouts,
                     uint32_t n_layers, uint64_t batch_seed, uint64_t* ids, uint64_t ids_cap,
                     uint64_t* n_ids, uint32_t* edges, uint64_t edges_cap,
                     uint64_t* layer_counts, uint64_t* io) {
    if (n_seeds == 0) return GXO_INVALID_ARGUMENT; /* sampler.hpp:72 */
    hmap h;
    hm_init(&h, 1024);
    uint64_t nid = 0, ne = 0;
    int rc = GXO_OK;
    uint32_t got;
    for (uint64_t i = 0; i < n_seeds; ++i) { /* sampler.hpp:80-85 */
        if (seeds[i] >= n_nodes) { rc = GXO_OUT_OF_RANGE; goto done; }
        if (!hm_emplace(&h, seeds[i], (uint32_t)nid, &got)) { rc = GXO_INVALID_ARGUMENT; goto done; }
        if (nid >= ids_cap) { rc = GXO_RUNTIME_ERROR; goto done; }
        ids[nid++] = seeds[i];
    }
    {
        sm64 r = {batch_seed};
        uint64_t scratch_cap = 16;
        uint64_t* scratch = (uint64_t*)malloc(scratch_cap * 8);
        for (uint32_t l = 0; l < n_layers; ++l) { /* sampler.hpp:89-115 */
            uint64_t frontier = nid;
            uint64_t le = 0;
            for (uint64_t k = 0; k < frontier; ++k) {
                uint64_t p = ids[k];
                uint64_t lo = indptr[p], hi = indptr[p + 1], deg = hi - lo;
                io[2] += 1;
                io[0] += gxo_pages_touched(8 * lo, 8 * hi);
                io[3] += 8 * deg;
                if (deg > scratch_cap) {
                    while (scratch_cap < deg) scratch_cap *= 2;
                    scratch = (uint64_t*)realloc(scratch, scratch_cap * 8);
                }
                memcpy(scratch, indices + lo, deg * 8);
                uint64_t take = fanouts[l] < deg ? fanouts[l] : deg;
                for (uint64_t j = 0; j < take; ++j) {
                    uint64_t pick = j + sm_bounded(&r, deg - j);
                    uint64_t t = scratch[j];
                    scratch[j] = scratch[pick];
                    scratch[pick] = t;
                    uint64_t child = scratch[j];
                    if (hm_emplace(&h, child, (uint32_t)nid, &got)) {
                        if (nid >= ids_cap) { free(scratch); rc = GXO_RUNTIME_ERROR; goto done; }
                        ids[nid++] = child;
                    }
                    if (ne >= edges_cap) { free(scratch); rc = GXO_RUNTIME_ERROR; goto done; }
                    edges[2 * ne] = got;
                    edges[2 * ne + 1] = (uint32_t)k;
                    ++ne;
                    ++le;
                }
            }
            layer_counts[l] = le;
        }
        free(scratch);
    }
done:
    *n_ids = nid;
    free(h.keys);
    free(h.vals);
    return rc;
}

/* ---- inspector: changeset.hpp ------------------------------------------ */
/* build_access_index (changeset.hpp:76-129). trace = S lists, flat + off[S+1].
 * iters_out: A+1 entries; ptr_out: N entries. */
int gxo_access_index(const uint64_t* flat, const uint64_t* off, uint64_t S, uint64_t N,
                     uint64_t* iters, uint64_t* ptr) {
    uint64_t* counts = (uint64_t*)calloc(N ? N : 1, 8);
    uint64_t* stamp = (uint64_t*)malloc((N ? N : 1) * 8);
    memset(stamp, 0xff, (N ? N : 1) * 8);
    int rc = GXO_OK;
    for (uint64_t i = 0; i < S; ++i) /* count_pass :76-88 */
        for (uint64_t a = off[i]; a < off[i + 1]; ++a) {
            uint64_t v = flat[a];
            if (v >= N) { rc = GXO_OUT_OF_RANGE; goto out; }
            if (stamp[v] == i) { rc = GXO_LOGIC_ERROR; goto out; }
            stamp[v] = i;
            counts[v]++;
        }
    { /* build_ptr :91-99, build_iters :104-122 */
        uint64_t acc = 0;
        for (uint64_t v = 0; v < N; ++v) {
            ptr[v] = acc;
            acc += counts[v];
        }
        uint64_t* cur = stamp; /* reuse */
        memcpy(cur, ptr, N * 8);
        for (uint64_t i = 0; i < S; ++i)
            for (uint64_t a = off[i]; a < off[i + 1]; ++a) iters[cur[flat[a]]++] = i;
        iters[acc] = ITER_DUMMY;
        for (uint64_t v = 0; v < N; ++v)
            if (counts[v]) iters[ptr[v]] |= ITER_FLAG;
    }
out:
    free(counts);
    free(stamp);
    return rc;
}

/* compute_init_set (changeset.hpp:137-153). */
int gxo_compute_init_set(const uint64_t* flat, const uint64_t* off, uint64_t S, uint64_t K,
                         uint64_t N, uint64_t* out, uint64_t* n_out) {
    *n_out = 0;
    if (K == 0) return GXO_OK;
    uint8_t* seen = (uint8_t*)calloc(N ? N : 1, 1);
    uint64_t n = 0;
    int rc = GXO_OK;
    for (uint64_t i = 0; i < S && n < K; ++i)
        for (uint64_t a = off[i]; a < off[i + 1]; ++a) {
            uint64_t v = flat[a];
            if (v >= N) { rc = GXO_OUT_OF_RANGE; goto out; }
            if (seen[v]) continue;
            seen[v] = 1;
            out[n++] = v;
            if (n == K) break;
        }
out:
    *n_out = n;
    free(seen);
    return rc;
}

typedef struct {
    uint64_t key;
    uint64_t is_new;
    uint64_t id;
    uint64_t pos;
} cand_t;
static int cand_cmp(const void* x, const void* y) { /* candidate_before, changeset.hpp:189-193 */
    const cand_t* a = (const cand_t*)x;
    const cand_t* b = (const cand_t*)y;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    if (a->is_new != b->is_new) return a->is_new < b->is_new ? -1 : 1;
    return a->id < b->id ? -1 : a->id > b->id;
}
static int pair_cmp(const void* x, const void* y) {
    const uint64_t* a = (const uint64_t*)x;
    const uint64_t* b = (const uint64_t*)y;
    if (a[0] != b[0]) return a[0] < b[0] ? -1 : 1;
    return a[1] < b[1] ? -1 : a[1] > b[1];
}

/* simulate_changesets (changeset.hpp:228-295) with finish_selection
 * (:198-220). Next accesses come from the AccessIndex exactly as the
 * reference walks it (cursor per node, parked on the dummy).
 * Outputs: misses[S]; in_ids/in_pos + in_off[S+1]; out_ids + out_off[S+1];
 * optionally the sorted state after each iteration (state/state_off). */
int gxo_simulate(const uint64_t* flat, const uint64_t* off, uint64_t S, uint64_t N, uint64_t K,
                 const uint64_t* init, uint64_t n_init, uint64_t* misses, uint64_t* in_ids,
                 uint64_t* in_pos, uint64_t* in_off, uint64_t* out_ids, uint64_t* out_off,
                 uint64_t* state_out, uint64_t* state_off, uint64_t state_cap) {
    uint64_t A = off[S];
    uint64_t* iters = (uint64_t*)malloc((A + 1) * 8);
    uint64_t* ptr = (uint64_t*)malloc((N ? N : 1) * 8);
    int rc = gxo_access_index(flat, off, S, N, iters, ptr);
    if (rc) { free(iters); free(ptr); return rc; }
    uint64_t* cursor = ptr; /* cursor starts at ptr (changeset.hpp:233) */
    uint8_t* resident = (uint8_t*)calloc(N ? N : 1, 1);
    uint64_t* state = (uint64_t*)malloc((K + n_init + 1) * 8);
    uint64_t ns = 0;
    cand_t* cand = NULL;
    uint64_t* incoming = NULL;
    uint64_t ki = 0, ko = 0, kst = 0;
    /* access_count(v) > 0  <=>  iters[ptr[v]] is a flagged region start of v;
     * keep the per-node counts to restate it exactly. */
    uint64_t* cnt = (uint64_t*)calloc(N ? N : 1, 8);
    for (uint64_t a = 0; a < A; ++a) cnt[flat[a]]++;
    for (uint64_t k = 0; k < n_init; ++k) { /* :238-247 */
        uint64_t v = init[k];
        if (v >= N) { rc = GXO_OUT_OF_RANGE; goto out; }
        if (cnt[v] == 0) { rc = GXO_LOGIC_ERROR; goto out; }
        if (resident[v]) { rc = GXO_LOGIC_ERROR; goto out; }
        resident[v] = 1;
        state[ns++] = v;
    }
    if (ns > K) { rc = GXO_INVALID_ARGUMENT; goto out; } /* :246 */
    qsort(state, ns, 8, cmp_u64);
    in_off[0] = 0;
    out_off[0] = 0;
    if (state_off) state_off[0] = 0;
    {
        uint64_t maxw = 0;
        for (uint64_t i = 0; i < S; ++i)
            if (off[i + 1] - off[i] > maxw) maxw = off[i + 1] - off[i];
        cand = (cand_t*)malloc((K + maxw + 1) * sizeof(cand_t));
        incoming = (uint64_t*)malloc((maxw + 1) * 16);
    }
    for (uint64_t i = 0; i < S; ++i) { /* :254-293 */
        uint64_t miss = 0;
        for (uint64_t a = off[i]; a < off[i + 1]; ++a) {
            uint64_t v = flat[a];
            if (!resident[v]) ++miss;
            uint64_t c = cursor[v] + 1;
            cursor[v] = (iters[c] & ITER_FLAG) ? A : c;
        }
        misses[i] = miss;
        uint64_t nc = 0;
        for (uint64_t s = 0; s < ns; ++s) {
            cand[nc].key = iters[cursor[state[s]]] & ITER_MASK;
            cand[nc].is_new = 0;
            cand[nc].id = state[s];
            cand[nc].pos = 0;
            nc++;
        }
        for (uint64_t a = off[i]; a < off[i + 1]; ++a) {
            uint64_t v = flat[a];
            if (!resident[v]) {
                cand[nc].key = iters[cursor[v]] & ITER_MASK;
                cand[nc].is_new = 1;
                cand[nc].id = v;
                cand[nc].pos = a - off[i];
                nc++;
            }
        }
        uint64_t keep = K < nc ? K : nc;
        qsort(cand, nc, sizeof(cand_t), cand_cmp); /* full order == nth_element prefix set */
        /* finish_selection :198-220 */
        uint64_t ninc = 0, o0 = ko;
        ns = 0;
        for (uint64_t k = 0; k < keep; ++k) {
            state[ns++] = cand[k].id;
            if (cand[k].is_new) {
                incoming[2 * ninc] = cand[k].pos;
                incoming[2 * ninc + 1] = cand[k].id;
                ninc++;
            }
        }
        for (uint64_t k = keep; k < nc; ++k)
            if (!cand[k].is_new) out_ids[ko++] = cand[k].id;
        qsort(incoming, ninc, 16, pair_cmp);
        for (uint64_t k = 0; k < ninc; ++k) {
            in_pos[ki] = incoming[2 * k];
            in_ids[ki] = incoming[2 * k + 1];
            ki++;
        }
        qsort(out_ids + o0, ko - o0, 8, cmp_u64);
        qsort(state, ns, 8, cmp_u64);
        for (uint64_t k = o0; k < ko; ++k) resident[out_ids[k]] = 0;
        for (uint64_t k = in_off[i]; k < ki; ++k) resident[in_ids[k]] = 1;
        in_off[i + 1] = ki;
        out_off[i + 1] = ko;
        if (state_out) {
            if (kst + ns > state_cap) { rc = GXO_RUNTIME_ERROR; goto out; }
            memcpy(state_out + kst, state, ns * 8);
            kst += ns;
            state_off[i + 1] = kst;
        }
    }
out:
    free(iters);
    free(ptr);
    free(resident);
    free(state);
    free(cand);
    free(incoming);
    free(cnt);
    return rc;
}

/* ---- executor: feature_cache.hpp:19-130 over an in-memory row table ------ */
typedef struct {
    uint64_t n_nodes, K;
    uint32_t row_bytes;
    const uint8_t* store; /* n_nodes rows of row_bytes (the features.bin payload) */
    int64_t* table;       /* address table, -1 = miss */
    uint8_t* rows;        /* K slots */
    uint64_t* free_slots; /* back = next slot handed out */
    uint64_t n_free;
} gxo_cache;

int gxo_cache_create(const uint8_t* store, uint64_t n_nodes, uint32_t row_bytes,
                     const uint64_t* init, uint64_t n_init, uint64_t K, uint64_t* io,
                     gxo_cache** out) {
    if (n_init > K) return GXO_INVALID_ARGUMENT; /* :22-23 */
    gxo_cache* c = (gxo_cache*)calloc(1, sizeof(gxo_cache));
    c->n_nodes = n_nodes;
    c->K = K;
    c->row_bytes = row_bytes;
    c->store = store;
    c->table = (int64_t*)malloc((n_nodes ? n_nodes : 1) * 8);
    memset(c->table, 0xff, (n_nodes ? n_nodes : 1) * 8);
    c->rows = (uint8_t*)malloc(K * row_bytes + 1);
    c->free_slots = (uint64_t*)malloc((K + 1) * 8);
    c->n_free = 0;
    for (uint64_t s = K; s > n_init; --s) c->free_slots[c->n_free++] = s - 1; /* :27-28 */
    for (uint64_t k = 0; k < n_init; ++k) {
        uint64_t v = init[k];
        int rc = 0;
        if (v >= n_nodes) rc = GXO_OUT_OF_RANGE;
        else if (c->table[v] >= 0) rc = GXO_INVALID_ARGUMENT;
        if (rc) {
            free(c->table); free(c->rows); free(c->free_slots); free(c);
            return rc;
        }
        memcpy(c->rows + k * row_bytes, store + v * row_bytes, row_bytes);
        io[1] += 1;
        io[0] += gxo_page_count_for_row(row_bytes, v);
        io[3] += row_bytes;
        c->table[v] = (int64_t)k;
    }
    *out = c;
    return GXO_OK;
}
void gxo_cache_destroy(gxo_cache* c) {
    if (!c) return;
    free(c->table);
    free(c->rows);
    free(c->free_slots);
    free(c);
}
int64_t gxo_cache_slot(const gxo_cache* c, uint64_t v) { return v < c->n_nodes ? c->table[v] : -1; }
const uint8_t* gxo_cache_row(const gxo_cache* c, uint64_t slot) { return c->rows + slot * c->row_bytes; }

/* gather (feature_cache.hpp:58-76): hits copy the slot, misses read the
 * store and are charged one row, page_count_for_row pages, row_bytes bytes. */
int gxo_cache_gather(const gxo_cache* c, const uint64_t* ids, uint64_t n, uint8_t* out,
                     uint64_t* hits, uint64_t* misses, uint64_t* io) {
    uint64_t h = 0, m = 0;
    const uint32_t w = c->row_bytes;
    for (uint64_t k = 0; k < n; ++k) {
        uint64_t v = ids[k];
        if (v >= c->n_nodes) return GXO_OUT_OF_RANGE;
        int64_t s = c->table[v];
        if (s >= 0) {
            if (out) memcpy(out + k * w, c->rows + (uint64_t)s * w, w);
            h++;
        } else {
            if (out) memcpy(out + k * w, c->store + v * w, w);
            m++;
            io[1] += 1;
            io[0] += gxo_page_count_for_row(w, v);
            io[3] += w;
        }
    }
    *hits = h;
    *misses = m;
    return GXO_OK;
}

/* apply_changeset (feature_cache.hpp:89-130): validate everything first, then
 * free out slots (out_ids order), fill in_ids[k] into freed[k] or pop the
 * free list, copy the row from batch[in_pos[k]], push back surplus. */
int gxo_cache_apply(gxo_cache* c, const uint8_t* batch, uint64_t rows, const uint64_t* ids,
                    uint64_t n_ids, const uint64_t* in_ids, const uint64_t* in_pos,
                    uint64_t n_in, const uint64_t* out_ids, uint64_t n_out) {
    if (rows != n_ids) return GXO_INVALID_ARGUMENT;
    for (uint64_t k = 0; k < n_in; ++k) {
        uint64_t v = in_ids[k], p = in_pos[k];
        if (p >= n_ids || ids[p] != v) return GXO_LOGIC_ERROR;
        if (v >= c->n_nodes) return GXO_OUT_OF_RANGE; /* reference indexes the table unchecked */
        if (c->table[v] >= 0) return GXO_LOGIC_ERROR;
    }
    for (uint64_t k = 0; k < n_out; ++k) {
        uint64_t v = out_ids[k];
        if (v >= c->n_nodes || c->table[v] < 0) return GXO_LOGIC_ERROR;
    }
    if (n_in > n_out + c->n_free) return GXO_LOGIC_ERROR;
    uint64_t* freed = (uint64_t*)malloc((n_out + 1) * 8);
    for (uint64_t k = 0; k < n_out; ++k) freed[k] = (uint64_t)c->table[out_ids[k]];
    for (uint64_t k = 0; k < n_out; ++k) c->table[out_ids[k]] = -1;
    const uint32_t w = c->row_bytes;
    for (uint64_t k = 0; k < n_in; ++k) {
        uint64_t slot = k < n_out ? freed[k] : c->free_slots[--c->n_free];
        memcpy(c->rows + slot * w, batch + in_pos[k] * w, w);
        c->table[in_ids[k]] = (int64_t)slot;
    }
    for (uint64_t k = n_in; k < n_out; ++k) c->free_slots[c->n_free++] = freed[k];
    free(freed);
    return GXO_OK;
}

uint64_t gxo_cache_resident(const gxo_cache* c, uint64_t* out) {
    uint64_t n = 0;
    for (uint64_t v = 0; v < c->n_nodes; ++v)
        if (c->table[v] >= 0) out[n++] = v;
    return n;
}

/* ---- compute_stub (pipeline.hpp:35-57): FNV-1a 64 over rows count, the row
 * bytes, the layer count, then per layer its edge count and (src, dst) u32
 * pairs -- the per-iteration checksum of TrainingRunner (pipeline.hpp:426). */
static void fnv_absorb(uint64_t* h, const void* p, uint64_t n) {
    const unsigned char* b = (const unsigned char*)p;
    for (uint64_t i = 0; i < n; ++i) {
        *h ^= b[i];
        *h *= 0x100000001B3ULL;
    }
}

uint64_t gxo_compute_stub(const void* rows, uint64_t n_rows, uint64_t row_bytes, const uint32_t* pairs,
                          const uint64_t* layer_counts, uint32_t n_layers) {
    uint64_t h = 0xCBF29CE484222325ULL;
    uint64_t v = n_rows;
    fnv_absorb(&h, &v, 8);
    fnv_absorb(&h, rows, n_rows * row_bytes);
    v = n_layers;
    fnv_absorb(&h, &v, 8);
    uint64_t k = 0;
    for (uint32_t l = 0; l < n_layers; ++l) {
        v = layer_counts[l];
        fnv_absorb(&h, &v, 8);
        fnv_absorb(&h, pairs + 2 * k, layer_counts[l] * 8);
        k += layer_counts[l];
    }
    return h;
}
