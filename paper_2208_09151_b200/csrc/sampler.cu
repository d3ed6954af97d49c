// sampler.cu -- multi-layer uniform neighbour sampling for a whole superbatch
// in ONE persistent, cooperatively launched kernel (all CTAs co-resident,
// phases separated by grid barriers).
//
// Reference: sample_batch (sampler.hpp:69-117) and superbatch_sample
// (sampler.hpp:197-243). Output is bit-identical:
//  * RNG: SplitMix64 per batch seeded derive_seed(global_seed, first+i)
//    (sampler.hpp:216). Draw t of the sequential stream == mix64(seed+t*gamma),
//    so the counter of draw j of parent k at layer l is
//        base_l + excl_scan_k(min(f_l, deg)) + j
//    and every draw is computed independently.
//  * Partial Fisher-Yates (sampler.hpp:103-107) on a FRESH copy of the sorted
//    in-list per parent. Picks are data-independent; the swap chain is
//    resolved on positions, so only the <= f chosen indices[] entries are read
//    and lists are never copied (resolve_pos below).
//  * Discovery-order dedup (sampler.hpp:78-84,108-112): per-batch open-address
//    table keyed by node id; a candidate child stores (NEW | flat draw
//    position) and 64-bit atomicMin keeps the first position; pre-existing ids
//    hold their local id (< NEW) and always win. Winners are ranked by draw
//    position (block scan + per-tile offsets), giving exactly the reference's
//    append order; edges are emitted in draw order.
//  * IoStats (graph_store.hpp:145-154): one list + pages_touched(8 ip[v],
//    8 ip[v+1]) + 8 deg bytes per expanded parent (no neighbor cache).
#include <algorithm>
#include <cooperative_groups.h>
#include <cstdlib>
#include <unordered_set>

#include "gx_internal.cuh"

namespace cg = cooperative_groups;

namespace gx {

constexpr int kMaxLayers = 16;
#ifndef GX_SB_THREADS
#define GX_SB_THREADS 256  // 256 x 4 CTAs/SM: 1.96 vs 2.00 ms (512 x 2), 1.98 (128 x 8), 2.14 (1024 x 1)
#endif
constexpr int SB_THREADS = GX_SB_THREADS;
#ifndef GX_SB_IPT
#define GX_SB_IPT 1  // parents per thread per tile (512-parent tiles: 2.00 vs 2.11 ms against 2)
#endif
constexpr int SB_IPT = GX_SB_IPT;
#ifndef GX_E_UNROLL
#define GX_E_UNROLL 2  // draws in flight per thread in phase E (round 1: 3 best of 2-6; with the tables sized by draws 2 is: 1.758 vs 1.770 ms, 4: 1.808, r02z_ab_sampler_e.txt)
#endif
#ifndef GX_TABLE_SLACK  // table slots >= entry bound << SLACK (1: load <= 1/2)
#define GX_TABLE_SLACK 1
#endif
#ifndef GX_TABLE_BY_DRAWS
#define GX_TABLE_BY_DRAWS 1
#endif
#ifndef GX_I_UNROLL
#define GX_I_UNROLL 4
#endif
#ifndef GX_E_LOADFIRST
#define GX_E_LOADFIRST 1
#endif
// 1024 threads per SM at 64 registers (a few spills): twice the warps of the
// 128-register build to hide the dependent random reads (measured 2.60 vs
// 2.86 ms per papers superbatch), split into four 256-thread CTAs.
#ifndef GX_SB_MINB
#define GX_SB_MINB (1024 / GX_SB_THREADS)
#endif
#define GX_SB_BOUNDS __launch_bounds__(SB_THREADS, GX_SB_MINB)
constexpr uint32_t SB_TILE = SB_THREADS * SB_IPT;
// draws per thread in the per-draw tile phases F and H (more independent
// loads in flight per thread than the per-parent tiles of A/E)
#ifndef GX_SB_DIPT
#define GX_SB_DIPT 4
#endif
constexpr int SB_DIPT = GX_SB_DIPT;
constexpr uint32_t SB_DTILE = SB_THREADS * SB_DIPT;
// F/H move a thread's SB_DIPT = 4 consecutive draws as 16-byte words (dslot,
// drank: one uint4; edges: two uint4) -- the per-batch draw / edge regions are
// padded to multiples of 4 draws so these are aligned and stay inside the
// region (GX_SB_VEC=0: the scalar per-draw form, 4 words per warp sector)
#ifndef GX_SB_VEC
#define GX_SB_VEC 1
#endif
static_assert(!GX_SB_VEC || SB_DIPT == 4, "vectorised F/H phases move 4 draws per thread");
constexpr uint32_t kNewBit = 0x80000000u;
constexpr unsigned long long kEmptySlot = ~0ull;
// batches per launch cap: sizes SampSmem's prefix arrays, and a small SampSmem
// leaves the SM's unified L1/shared array to L1 (spills, read-only loads)
constexpr uint32_t kMaxBatchesPerLaunch = 512;
constexpr uint64_t kChunk = 128;  // batches per sampler launch
constexpr int kPickCache = 32;

struct SampArgs {
    const uint64_t* __restrict__ indptr;
    const uint32_t* __restrict__ indices;
    // row-partitioned CSC (nparts > 0): edge e of rank q's range lives at
    // part[q][e - ebound[q]] -- this rank's HBM or a peer's over NVLink (IPC)
    uint32_t nparts;
    const uint32_t* part[kMaxParts];
    uint64_t ebound[kMaxParts + 1];
    uint64_t N;
    uint32_t S, L;
    uint32_t fan[kMaxLayers];
    const uint64_t* bseed;
    const uint32_t* seeds;
    const uint64_t* seed_off;
    uint32_t* ids;
    uint64_t cap_ids;
    uint32_t* n_ids;
    uint2* edges;
    uint64_t cap_e_batch;
    uint64_t e_off[kMaxLayers];
    uint32_t* layer_count;
    uint32_t* F;
    uint32_t* T;
    uint64_t* dbase;
    uint32_t* pscan;
    uint64_t* plo;
    uint32_t* pdeg;
    uint32_t* idslot;
    uint32_t* tsum;
    uint32_t* tsum2;
    uint32_t* dslot;
    uint32_t* drank;
    uint64_t cap_draw;
    unsigned long long* tab0;
    unsigned long long* tab1;
    uint64_t tab_cap;  // per batch max
    unsigned long long* io;
    const uint32_t* ncbits;     // neighbor cache: a cached list charges no I/O (sampler.hpp:91-97)
    // the inspector's first-use array, filled as ids are discovered (pipeline):
    // firstx[v] = max(firstx[v], fx_epoch - ((batch0 + b) << 21 | local))
    uint32_t* firstx;
    uint32_t fx_epoch, batch0;
    GridBarrier* bar;
    uint32_t* tctr;             // dynamic tile counters, 4 per layer (zeroed at kernel start)
    // phase E stages a tile's (position, parent) draws in shared memory (after
    // SampSmem, SB_TILE x max fanout entries) instead of the edge slots, so the
    // draw loop's first load is an smem read, not an L2 round trip
    uint32_t stage_smem;
    unsigned long long* trace;  // optional phase timestamps (GX_SAMPLER_TRACE)
};

#define TRACE_STAMP(a, l, ph)                                                  \
    do {                                                                       \
        if ((a).trace && blockIdx.x == 0 && threadIdx.x == 0)                  \
            (a).trace[1 + (l) * 8 + (ph)] = gtimer() - (a).trace[0];           \
    } while (0)

// indices[e]: the whole CSC, or the owner's partition (peer loads over NVLink
// fuse the per-layer request/response exchange of sampler.hpp:89-115 into the
// draw loop; every index in the parameter bank is static, no local copies)
__device__ __forceinline__ uint32_t ld_index(const SampArgs& a, uint64_t e) {
    if (a.nparts == 0) return __ldg(a.indices + e);
    const uint32_t* base = a.part[0];
    uint64_t lo = 0;
#pragma unroll
    for (int q = 1; q < kMaxParts; ++q)
        if (q < (int)a.nparts && e >= a.ebound[q]) {
            base = a.part[q];
            lo = a.ebound[q];
        }
    return __ldg(base + (e - lo));
}

struct SampSmem {
    uint32_t scan[34];
    unsigned long long red[34];
    uint32_t tp[kMaxBatchesPerLaunch + 1];
    uint32_t px[kMaxBatchesPerLaunch + 1];  // raw per-batch item prefix (flattened loops)
    unsigned long long plo_s[SB_TILE];      // phase E: list offsets of the tile's parents
    uint32_t tnext;                         // dynamically scheduled tile (broadcast)
};

// px[0..S] = prefix of per-batch item counts (seeds of batch b when
// seed_off != nullptr, else cnt[b]); returns the total. Lets a phase spread
// (batch, item) pairs over the whole grid instead of looping batch by batch.
__device__ uint32_t build_prefix(const uint32_t* cnt, const uint64_t* seed_off, uint32_t S, SampSmem& sm) {
    uint32_t carry = 0;
    for (uint32_t base = 0; base < S; base += blockDim.x) {
        const uint32_t b = base + threadIdx.x;
        uint32_t v = 0;
        if (b < S) v = seed_off ? (uint32_t)(seed_off[b + 1] - seed_off[b]) : cnt[b];
        uint32_t tot;
        const uint32_t ex = block_excl_scan(v, sm.scan, tot);
        if (b < S) sm.px[b] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) sm.px[S] = carry;
    __syncthreads();
    return carry;
}
__device__ __forceinline__ uint32_t prefix_batch(const SampSmem& sm, uint32_t S, uint32_t x) {
    uint32_t lo = 0, hi = S;  // b: px[b] <= x < px[b+1]
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (sm.px[mid] <= x) lo = mid;
        else hi = mid;
    }
    return lo;
}

// tp[0..S] = prefix of ceil(cnt[b] / TILE); returns total tiles.
template <uint32_t TILE = SB_TILE>
__device__ uint32_t build_tiles(const uint32_t* cnt, uint32_t S, SampSmem& sm) {
    uint32_t carry = 0;
    for (uint32_t base = 0; base < S; base += blockDim.x) {
        uint32_t b = base + threadIdx.x;
        uint32_t v = b < S ? (cnt[b] + TILE - 1) / TILE : 0;
        uint32_t tot;
        uint32_t ex = block_excl_scan(v, sm.scan, tot);
        if (b < S) sm.tp[b] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) sm.tp[S] = carry;
    __syncthreads();
    return carry;
}

__device__ __forceinline__ uint32_t tile_batch(const SampSmem& sm, uint32_t S, uint32_t t) {
    uint32_t lo = 0, hi = S;  // find b: tp[b] <= t < tp[b+1]
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (sm.tp[mid] <= t) lo = mid;
        else hi = mid;
    }
    return lo;
}

// Sum of tile sums of batch b's tiles before tile t (one warp; result to all threads).
__device__ __forceinline__ uint32_t tile_offset(const uint32_t* tsum, uint32_t first, uint32_t t,
                                                uint32_t* bcast) {
    if (threadIdx.x < 32) {
        uint32_t s = 0;
        for (uint32_t i = first + threadIdx.x; i < t; i += 32) s += tsum[i];
        s = warp_sum(s);
        if (threadIdx.x == 0) *bcast = s;
    }
    __syncthreads();
    uint32_t r = *bcast;
    __syncthreads();
    return r;
}

// *dup (optional) is set when the key was already present: at layer 0 that
// is a duplicate seed, which the reference rejects (sampler.hpp:83)
__device__ __forceinline__ uint32_t table_insert(unsigned long long* tab, uint32_t H, uint32_t key,
                                                 uint32_t val, bool* dup = nullptr) {
    const unsigned long long ent = ((unsigned long long)key << 32) | val;
    uint32_t s = hash32(key) & (H - 1);
    while (true) {
        unsigned long long cur = __ldcg(tab + s);  // never trust a stale L1 line
        if (cur == kEmptySlot) {
            unsigned long long prev = atomicCAS(&tab[s], kEmptySlot, ent);
            if (prev == kEmptySlot) return s;
            cur = prev;
        }
        if ((uint32_t)(cur >> 32) == key) {
            if (cur > ent) atomicMin(&tab[s], ent);
            if (dup) *dup = true;
            return s;
        }
        s = (s + 1) & (H - 1);
    }
}

// Insert for a draw: CAS first (one round trip when the slot is free).
// *prior = the key's value before this insert: a local id (< kNewBit) when the
// child was already in ids -- final for this layer, so the edge resolves now --
// else kEmpty32 / another draw's (NEW | position).
constexpr uint32_t kResolved = 0x80000000u;  // dslot flag: edge source known at insert time
__device__ __forceinline__ uint32_t table_insert_draw(unsigned long long* tab, uint32_t H, uint32_t key,
                                                      uint32_t val, uint32_t* prior) {
    const unsigned long long ent = ((unsigned long long)key << 32) | val;
    uint32_t s = hash32(key) & (H - 1);
    while (true) {
        const unsigned long long cur = atomicCAS(&tab[s], kEmptySlot, ent);
        if (cur == kEmptySlot) {
            *prior = kEmpty32;
            return s;
        }
        if ((uint32_t)(cur >> 32) == key) {
            if (cur > ent) atomicMin(&tab[s], ent);
            *prior = (uint32_t)cur;
            return s;
        }
        s = (s + 1) & (H - 1);
    }
}

__device__ __forceinline__ uint32_t pick_at(uint64_t seed, uint64_t t0, uint32_t i, uint32_t deg) {
    return i + (uint32_t)draw_bounded(seed, t0 + i, (uint64_t)(deg - i));
}

// Position (within the parent's sorted list) of the child taken at FY step j:
// P_j[pick_j], where P_j[x] = P_i[i] for the latest i < j with pick_i == x,
// else x (sampler.hpp:103-107 resolved without materialising the list).
__device__ __forceinline__ uint32_t resolve_pos(const uint32_t* pk, uint32_t j, uint64_t seed,
                                                uint64_t t0, uint32_t deg) {
    uint32_t c = pk[j < kPickCache ? j : 0];
    if (j >= kPickCache) c = pick_at(seed, t0, j, deg);
    uint32_t lim = j;
    while (true) {
        int found = -1;
        for (int i = (int)lim - 1; i >= 0; --i) {
            uint32_t pi = i < kPickCache ? pk[i] : pick_at(seed, t0, (uint32_t)i, deg);
            if (pi == c) {
                found = i;
                break;
            }
        }
        if (found < 0) return c;
        c = (uint32_t)found;
        lim = (uint32_t)found;
    }
}

// Positions of a parent's tk draws (partial Fisher-Yates, sampler.hpp:103-107)
// written as (position, parent) into out[0..tk). Fast path (tk <= 16): picks in
// registers; a 64-bit filter over the low pick bits proves most picks
// collision-free (then the child sits at the picked position), the rest
// resolve the swap chain exactly over the register array.
__device__ __forceinline__ void draw_positions(uint32_t tk, uint64_t seed, uint64_t t0, uint32_t deg,
                                               uint2* out, uint32_t parent) {
    constexpr int MAXT = 16;
    if (tk <= MAXT) {
        uint32_t pk[MAXT];
#pragma unroll
        for (int q = 0; q < MAXT; ++q) pk[q] = (uint32_t)q < tk ? pick_at(seed, t0, q, deg) : 0xFFFFFFFFu;
        unsigned long long filt = 0;
#pragma unroll
        for (int q = 0; q < MAXT; ++q) {
            if ((uint32_t)q < tk) {
                uint32_t c = pk[q];
                const unsigned long long bit = 1ull << (c & 63);
                if (filt & bit) {
                    int lim = q;
                    while (true) {
                        int found = -1;
#pragma unroll
                        for (int i = 0; i < MAXT; ++i)
                            if (i < lim && pk[i] == c) found = i;  // latest i < lim
                        if (found < 0) break;
                        c = (uint32_t)found;
                        lim = found;
                    }
                }
                filt |= bit;
                out[q] = make_uint2(c, parent);
            }
        }
    } else {
        uint32_t pk[kPickCache];
        for (uint32_t q = 0; q < (uint32_t)kPickCache; ++q) pk[q] = pick_at(seed, t0, q, deg);
        for (uint32_t q = 0; q < tk; ++q) out[q] = make_uint2(resolve_pos(pk, q, seed, t0, deg), parent);
    }
}

// Clear the first H entries of each of the S per-batch tables (16-byte stores).
// phase F's per-draw word for an unresolved draw whose table entry is e: 1 for
// the winner (the entry holds this draw's position), 0 for a loser, or on the
// last layer kNewBit | the winner's position so phase I finds the winner's
// local id without re-reading the table (another random DRAM sector per loser)
__device__ __forceinline__ uint32_t loser_code(unsigned long long e, uint32_t child, uint32_t p, bool last) {
    if (e == (((unsigned long long)child << 32) | (kNewBit | p))) return 1u;
    return last ? (kNewBit | ((uint32_t)e & ~kNewBit)) : 0u;
}

__device__ __forceinline__ void clear_region(unsigned long long* tab, uint64_t tab_cap, uint32_t H, uint32_t S) {
    const uint64_t total_threads = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t per = H / 2;  // ulonglong2 per batch (H is a power of two >= 1024)
    const ulonglong2 e = make_ulonglong2(kEmptySlot, kEmptySlot);
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < (uint64_t)S * per; x += total_threads) {
        const uint64_t b = x / per, o = x - b * per;
        reinterpret_cast<ulonglong2*>(tab + b * tab_cap)[o] = e;
    }
}

__global__ void GX_SB_BOUNDS k_sample(SampArgs a) {
    extern __shared__ unsigned char smem_raw[];
    SampSmem& sm = *reinterpret_cast<SampSmem*>(smem_raw);
    uint2* const sm_stage = reinterpret_cast<uint2*>(smem_raw + ((sizeof(SampSmem) + 15) & ~size_t(15)));
    __shared__ uint32_t bcast;
    const uint32_t S = a.S;
    const uint32_t tid = threadIdx.x;
    int cur = 0;
    uint32_t H = 0;
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[0] = gtimer();
    // tile counters: first used after several grid barriers
    if (blockIdx.x == 0)
        for (uint32_t i = threadIdx.x; i < 4 * kMaxLayers; i += blockDim.x) a.tctr[i] = 0;

    for (uint32_t l = 0; l < a.L || l == 0; ++l) {
        // ---- Phase D: (re)build the per-batch tables with the current ids --
        // H = nextpow2(2 * max_b(entries bound)) keeps the load <= 1/2.
        auto phase_d = [&](bool by_draws) {
        uint32_t newH;
        {
            unsigned long long mx = 0;
            // entries the layer's table can hold: the ids so far plus at most
            // one per draw -- after phase A the draw count T_b is known (tile
            // sums of takes), before it (layer 0) bound it by F_b * f
            if (by_draws) build_tiles(a.F, S, sm);
            for (uint32_t b = tid; b < S; b += blockDim.x) {
                unsigned long long fb = l == 0 ? (a.seed_off[b + 1] - a.seed_off[b]) : a.F[b];
                unsigned long long need;
                if (by_draws) {
                    unsigned long long tb = 0;
                    for (uint32_t i = sm.tp[b]; i < sm.tp[b + 1]; ++i) tb += a.tsum[i];
                    need = fb + tb;
                } else {
                    need = fb * (1ull + (a.L ? a.fan[l] : 0));
                }
                mx = max(mx, need);
            }
            // block max via the scan buffer
            for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            if ((tid & 31) == 0) sm.red[tid >> 5] = mx;
            __syncthreads();
            if (tid == 0) {
                unsigned long long m = 0;
                for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = max(m, sm.red[w]);
                m = m < a.cap_ids ? m : (unsigned long long)a.cap_ids;
                unsigned long long h = 1024;
                while (h < (m << GX_TABLE_SLACK)) h <<= 1;
                if (h > a.tab_cap) h = a.tab_cap;
                sm.red[32] = h;
            }
            __syncthreads();
            newH = (uint32_t)sm.red[32];
            __syncthreads();
        }
        if (l == 0 || newH != H) {
            unsigned long long* told = cur ? a.tab1 : a.tab0;
            unsigned long long* tnew = cur ? a.tab0 : a.tab1;
            if (l == 0) tnew = told;  // tables start clean
            const uint64_t total_threads = (uint64_t)gridDim.x * blockDim.x;
            const uint32_t tot = build_prefix(a.F, l == 0 ? a.seed_off : nullptr, S, sm);
            for (uint32_t x = blockIdx.x * blockDim.x + tid; x < tot; x += (uint32_t)total_threads) {
                const uint32_t b = prefix_batch(sm, S, x);
                const uint32_t k = x - sm.px[b];
                const uint64_t gi = (uint64_t)b * a.cap_ids + k;
                uint32_t v;
                if (l == 0) {
                    v = a.seeds[a.seed_off[b] + k];
                    a.ids[gi] = v;
                    if (a.firstx) atomicMax(&a.firstx[v], a.fx_epoch - (((a.batch0 + b) << 21) | k));
                } else {
                    v = a.ids[gi];
                }
                bool dup = false;
                table_insert(tnew + (uint64_t)b * a.tab_cap, newH, v, k, l == 0 ? &dup : nullptr);
                if (dup) atomicOr(&a.io[3], 1ull);  // duplicate seed: the host fails the call
            }
            if (l > 0) {  // the previous layer's table is dead: bulk-clear its used region
                clear_region(told, a.tab_cap, H, S);
                cur ^= 1;
            }
            H = newH;
            if (l == 0) {
                for (uint32_t b = blockIdx.x * blockDim.x + tid; b < S; b += total_threads) {
                    uint32_t ns = (uint32_t)(a.seed_off[b + 1] - a.seed_off[b]);
                    a.F[b] = ns;
                    a.n_ids[b] = ns;
                    a.dbase[b] = 0;
                }
            }
            grid_sync(a.bar);
            TRACE_STAMP(a, l, 0);
        }
        };
        // GX_TABLE_BY_DRAWS=1 (default) sizes layers >= 1 by the actual draw count
        // (phase A first): the last layer's tables are half as large (0.39 vs
        // 0.78 GB per papers superbatch, load <= 0.42). The sampler is bound by
        // random DRAM accesses, so the smaller footprint wins: k_sample 1.84 ->
        // 1.78 ms (2 A/B pairs, profiles/r02z_ab_table_by_draws.txt; round 1 had
        // measured it slower before the F/H vectorisation). Load ~0.7 (slack 0)
        // is far slower (2.80 ms): the probe chains grow. GX_TABLE_BY_DRAWS=0
        // sizes by F_b * (1 + f).
        if (l == 0 || !GX_TABLE_BY_DRAWS) phase_d(false);
        if (a.L == 0) break;
        const uint32_t f = a.fan[l];
        const bool last_layer = l + 1 == a.L;

        // ---- Phase A: per parent deg/take, IoStats, tile sums of takes ----
        {
            uint32_t ntiles = build_tiles(a.F, S, sm);
            unsigned long long io_pages = 0, io_lists = 0, io_bytes = 0;
            for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const uint32_t b = tile_batch(sm, S, t);
                const uint32_t Fb = a.F[b];
                const uint32_t k0 = (t - sm.tp[b]) * SB_TILE + tid * SB_IPT;
                uint32_t s = 0;
#pragma unroll
                for (int j = 0; j < SB_IPT; ++j) {
                    const uint32_t k = k0 + j;
                    if (k < Fb) {
                        const uint64_t gi = (uint64_t)b * a.cap_ids + k;
                        const uint32_t v = a.ids[gi];
                        const uint64_t lo = a.indptr[v], hi = a.indptr[v + 1];
                        const uint32_t deg = (uint32_t)(hi - lo);
                        const uint32_t take = min(f, deg);
                        a.plo[gi] = lo;
                        a.pdeg[gi] = deg;
                        a.pscan[gi] = take;
                        s += take;
                        if (!a.ncbits || !((__ldg(a.ncbits + (v >> 5)) >> (v & 31)) & 1u)) {
                            io_lists += 1;
                            io_pages += pages_touched(8 * lo, 8 * hi);
                            io_bytes += 8ull * deg;
                        }
                    }
                }
                uint32_t tot = block_sum(s, sm.scan);
                if (tid == 0) a.tsum[t] = tot;
            }
            io_pages = warp_sum(io_pages);
            io_lists = warp_sum(io_lists);
            io_bytes = warp_sum(io_bytes);
            if ((tid & 31) == 0 && io_lists) {
                atomicAdd(&a.io[0], io_pages);
                atomicAdd(&a.io[1], io_lists);
                atomicAdd(&a.io[2], io_bytes);
            }
        }
        grid_sync(a.bar);
        TRACE_STAMP(a, l, 1);

        if (l > 0 && GX_TABLE_BY_DRAWS) phase_d(true);
        unsigned long long* tab = cur ? a.tab1 : a.tab0;

        // ---- Phase E: scan takes -> draw offsets; draw, read child, insert ----
        {
            uint32_t ntiles = build_tiles(a.F, S, sm);
            // tiles carry very different draw counts: hand them out dynamically
            // (consecutive tiles -> the CTAs share a few batches' tables in L2)
            for (;;) {
                if (tid == 0) sm.tnext = atomicAdd(&a.tctr[4 * l], 1u);
                __syncthreads();
                const uint32_t t = sm.tnext;
                if (t >= ntiles) break;
                const uint32_t b = tile_batch(sm, S, t);
                const uint32_t Fb = a.F[b];
                const uint32_t first = sm.tp[b];
                const uint32_t toff = tile_offset(a.tsum, first, t, &bcast);
                if (t == first && tid < 32) {  // batch total T_b
                    uint32_t s2 = 0;
                    for (uint32_t i = first + tid; i < sm.tp[b + 1]; i += 32) s2 += a.tsum[i];
                    s2 = warp_sum(s2);
                    if (tid == 0) a.T[b] = s2;
                }
                const uint32_t k0 = (t - first) * SB_TILE + tid * SB_IPT;
                uint32_t take[SB_IPT];
                uint32_t s = 0;
#pragma unroll
                for (int j = 0; j < SB_IPT; ++j) {
                    const uint32_t k = k0 + j;
                    take[j] = k < Fb ? a.pscan[(uint64_t)b * a.cap_ids + k] : 0;
                    s += take[j];
                }
                uint32_t tot;
                uint32_t off = toff + block_excl_scan(s, sm.scan, tot);
                const uint64_t seed = a.bseed[b];
                const uint64_t dbase = a.dbase[b];
                unsigned long long* btab = tab + (uint64_t)b * a.tab_cap;
                uint2* bedge = a.edges + (uint64_t)b * a.cap_e_batch + a.e_off[l];
                uint32_t* bdslot = a.dslot + (uint64_t)b * a.cap_draw;
                const uint32_t d_begin = off;  // this thread's first draw
                long long c_e1 = 0;
                if (a.trace && tid == 0) c_e1 = clock64();
                // E1 (per parent, registers only): FY positions of every draw,
                // staged as (position, parent) in the edge slot; the parents'
                // list offsets go to shared memory for E2.
                for (int j = 0; j < SB_IPT; ++j) {
                    const uint32_t tk = take[j];
                    if (tk) {
                        const uint64_t gi = (uint64_t)b * a.cap_ids + k0 + j;
                        sm.plo_s[tid * SB_IPT + j] = a.plo[gi];
                        draw_positions(tk, seed, dbase + off, a.pdeg[gi],
                                       a.stage_smem ? sm_stage + (off - toff) : bedge + off, k0 + j);
                    }
                    off += tk;
                }
                (void)d_begin;
                __syncthreads();  // the tile's staged draws are visible to the whole CTA
                long long c_e2 = 0;
                if (a.trace && tid == 0 && l < 8) {
                    c_e2 = clock64();
                    atomicAdd(&a.trace[100 + 2 * l], (unsigned long long)(c_e2 - c_e1));
                }
                // E2 (per draw): child read, edge, dedup insert -- one draw per
                // thread so the random reads and atomics of a tile overlap.
                const uint32_t tile_d0 = toff, tile_d1 = toff + tot;
                const uint32_t tile_k0 = (t - first) * SB_TILE;  // the tile's first parent
                constexpr int U = GX_E_UNROLL;  // draws per thread in flight
                for (uint32_t q0 = tile_d0 + tid; q0 < tile_d1; q0 += U * blockDim.x) {
                    uint2 st[U];
                    uint32_t child[U];
#pragma unroll
                    for (int j = 0; j < U; ++j) {
                        const uint32_t p = q0 + j * blockDim.x;
                        if (p < tile_d1) st[j] = a.stage_smem ? sm_stage[p - tile_d0] : bedge[p];
                    }
#pragma unroll
                    for (int j = 0; j < U; ++j) {
                        const uint32_t p = q0 + j * blockDim.x;
                        if (p < tile_d1) child[j] = ld_index(a, sm.plo_s[st[j].y - tile_k0] + st[j].x);
                    }
                    // first probes of all U draws back to back, then resolve
                    uint32_t slot[U];
                    unsigned long long got[U];
#pragma unroll
                    for (int j = 0; j < U; ++j) {
                        const uint32_t p = q0 + j * blockDim.x;
                        if (p < tile_d1) {
                            slot[j] = hash32(child[j]) & (H - 1);
#if GX_E_LOADFIRST
                            got[j] = __ldcg(&btab[slot[j]]);
#else
                            got[j] = atomicCAS(&btab[slot[j]], kEmptySlot,
                                               ((unsigned long long)child[j] << 32) | (kNewBit | p));
#endif
                        }
                    }
#if GX_E_LOADFIRST
                    // claim the empty first slots (a match needs no CAS; most repeats of a hub stop here)
#pragma unroll
                    for (int j = 0; j < U; ++j) {
                        const uint32_t p = q0 + j * blockDim.x;
                        if (p < tile_d1 && got[j] == kEmptySlot)
                            got[j] = atomicCAS(&btab[slot[j]], kEmptySlot,
                                               ((unsigned long long)child[j] << 32) | (kNewBit | p));
                    }
#endif
#pragma unroll
                    for (int j = 0; j < U; ++j) {
                        const uint32_t p = q0 + j * blockDim.x;
                        if (p < tile_d1) {
                            const unsigned long long ent = ((unsigned long long)child[j] << 32) | (kNewBit | p);
                            uint32_t sl = slot[j], prior;
                            unsigned long long cur = got[j];
                            while (true) {
                                if (cur == kEmptySlot) {
                                    prior = kEmpty32;
                                    break;
                                }
                                if ((uint32_t)(cur >> 32) == child[j]) {
                                    if (cur > ent) atomicMin(&btab[sl], ent);
                                    prior = (uint32_t)cur;
                                    break;
                                }
                                sl = (sl + 1) & (H - 1);
                                cur = atomicCAS(&btab[sl], kEmptySlot, ent);
                            }
                            if (prior < kNewBit) {  // child already in ids: its local id is final
                                bedge[p] = make_uint2(prior, st[j].y);
                                bdslot[p] = sl | kResolved;
                            } else {
                                bedge[p] = make_uint2(child[j], st[j].y);
                                bdslot[p] = sl;
                            }
                        }
                    }
                }
                __syncthreads();
                if (a.trace && tid == 0 && l < 8)
                    atomicAdd(&a.trace[101 + 2 * l], (unsigned long long)(clock64() - c_e2));
            }
        }
        grid_sync(a.bar);
        TRACE_STAMP(a, l, 2);

        // ---- Phase F: first-occurrence flags per draw, tile sums ----------
        {
            uint32_t ntiles = build_tiles<SB_DTILE>(a.T, S, sm);
            for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const uint32_t b = tile_batch(sm, S, t);
                const uint32_t Tb = a.T[b];
                const uint32_t p0 = (t - sm.tp[b]) * SB_DTILE + tid * SB_DIPT;
                const unsigned long long* btab = tab + (uint64_t)b * a.tab_cap;
                const uint2* bedge = a.edges + (uint64_t)b * a.cap_e_batch + a.e_off[l];
                uint32_t s = 0;
#if GX_SB_VEC
                if (p0 < Tb) {
                    const uint64_t gd0 = (uint64_t)b * a.cap_draw + p0;
                    const uint4 d4 = *reinterpret_cast<const uint4*>(a.dslot + gd0);
                    const uint4 e01 = *reinterpret_cast<const uint4*>(bedge + p0);
                    const uint4 e23 = *reinterpret_cast<const uint4*>(bedge + p0 + 2);
                    const uint32_t ds[4] = {d4.x, d4.y, d4.z, d4.w}, ch[4] = {e01.x, e01.z, e23.x, e23.z};
                    uint32_t fl[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        fl[j] = 0;
                        if (p0 + j < Tb && !(ds[j] & kResolved)) {
                            const unsigned long long e = btab[ds[j]];
                            fl[j] = loser_code(e, ch[j], p0 + j, last_layer);
                        }
                        s += fl[j] == 1u;
                    }
                    *reinterpret_cast<uint4*>(a.drank + gd0) = make_uint4(fl[0], fl[1], fl[2], fl[3]);
                }
#else
#pragma unroll
                for (int j = 0; j < SB_DIPT; ++j) {
                    const uint32_t p = p0 + j;
                    if (p < Tb) {
                        const uint64_t gd = (uint64_t)b * a.cap_draw + p;
                        const uint32_t ds = a.dslot[gd];
                        uint32_t fl = 0;
                        if (!(ds & kResolved)) {
                            const unsigned long long e = btab[ds];
                            const uint32_t child = bedge[p].x;
                            fl = loser_code(e, child, p, last_layer);
                        }
                        a.drank[gd] = fl;
                        s += fl == 1u;
                    }
                }
#endif
                uint32_t tot = block_sum(s, sm.scan);
                if (tid == 0) a.tsum2[t] = tot;
            }
        }
        grid_sync(a.bar);
        TRACE_STAMP(a, l, 3);

        // ---- Phase H: rank winners by draw position -> new local ids -------
        {
            uint32_t ntiles = build_tiles<SB_DTILE>(a.T, S, sm);
            for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const uint32_t b = tile_batch(sm, S, t);
                const uint32_t Tb = a.T[b];
                const uint32_t first = sm.tp[b];
                const uint32_t Fb = a.F[b];
                const uint32_t toff = tile_offset(a.tsum2, first, t, &bcast);
                if (t == first && tid < 32) {
                    uint32_t s2 = 0;
                    for (uint32_t i = first + tid; i < sm.tp[b + 1]; i += 32) s2 += a.tsum2[i];
                    s2 = warp_sum(s2);
                    if (tid == 0) a.n_ids[b] = Fb + s2;
                }
                const uint32_t p0 = (t - first) * SB_DTILE + tid * SB_DIPT;
                uint32_t fl[SB_DIPT];
                uint32_t s = 0;
#if GX_SB_VEC
                const uint64_t gd0 = (uint64_t)b * a.cap_draw + p0;
                uint4 r4 = make_uint4(0, 0, 0, 0);
                if (p0 < Tb) r4 = *reinterpret_cast<const uint4*>(a.drank + gd0);
                fl[0] = r4.x == 1u;
                fl[1] = p0 + 1 < Tb && r4.y == 1u;
                fl[2] = p0 + 2 < Tb && r4.z == 1u;
                fl[3] = p0 + 3 < Tb && r4.w == 1u;
                s = fl[0] + fl[1] + fl[2] + fl[3];
#else
#pragma unroll
                for (int j = 0; j < SB_DIPT; ++j) {
                    const uint32_t p = p0 + j;
                    fl[j] = p < Tb && a.drank[(uint64_t)b * a.cap_draw + p] == 1u;
                    s += fl[j];
                }
#endif
                uint32_t tot;
                uint32_t r = toff + block_excl_scan(s, sm.scan, tot);
                unsigned long long* btab = tab + (uint64_t)b * a.tab_cap;
                uint2* bedge_w = a.edges + (uint64_t)b * a.cap_e_batch + a.e_off[l];
                const uint2* bedge = bedge_w;
#if GX_SB_VEC
                if (s) {  // winners: the thread's 4 edges (and rank words) rewritten as 16-byte words
                    uint4 e01 = *reinterpret_cast<const uint4*>(bedge + p0);
                    uint4 e23 = *reinterpret_cast<const uint4*>(bedge + p0 + 2);
                    uint32_t ch[4] = {e01.x, e01.z, e23.x, e23.z}, rk[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (fl[j]) {
                            const uint32_t child = ch[j];
                            const uint32_t local = Fb + r;
                            a.ids[(uint64_t)b * a.cap_ids + local] = child;
                            if (a.firstx)  // fire-and-forget: overlaps the latency-bound phases
                                atomicMax(&a.firstx[child], a.fx_epoch - (((a.batch0 + b) << 21) | local));
                            if (last_layer) {
                                rk[j] = local;  // phase I follows the table's winning position here
                            } else {
                                const uint32_t slot = a.dslot[gd0 + j];
                                btab[slot] = ((unsigned long long)child << 32) | local;
                            }
                            ch[j] = local;
                            ++r;
                        }
                    }
                    e01.x = ch[0];
                    e01.z = ch[1];
                    e23.x = ch[2];
                    e23.z = ch[3];
                    *reinterpret_cast<uint4*>(bedge_w + p0) = e01;
                    *reinterpret_cast<uint4*>(bedge_w + p0 + 2) = e23;
                    if (last_layer) *reinterpret_cast<uint4*>(a.drank + gd0) = make_uint4(rk[0], rk[1], rk[2], rk[3]);
                }
                if (false)
#endif
#pragma unroll
                for (int j = 0; j < SB_DIPT; ++j) {
                    if (fl[j]) {
                        const uint32_t p = p0 + j;
                        const uint32_t child = bedge[p].x;
                        const uint32_t local = Fb + r;
                        a.ids[(uint64_t)b * a.cap_ids + local] = child;
                        if (a.firstx)  // fire-and-forget: overlaps the latency-bound phases
                            atomicMax(&a.firstx[child], a.fx_epoch - (((a.batch0 + b) << 21) | local));
                        if (last_layer) {
                            // the table is never read again by node: the winner's
                            // local id goes to its own draw slot (coalesced), and
                            // phase I follows the table's winning position there
                            a.drank[(uint64_t)b * a.cap_draw + p] = local;
                        } else {
                            const uint32_t slot = a.dslot[(uint64_t)b * a.cap_draw + p];
                            btab[slot] = ((unsigned long long)child << 32) | local;
                        }
                        bedge_w[p].x = local;
                        ++r;
                    }
                }
            }
        }
        grid_sync(a.bar);
        TRACE_STAMP(a, l, 4);

        // ---- Phase I: edge sources -> local ids; per-batch bookkeeping ------
        {
            const uint64_t total_threads = (uint64_t)gridDim.x * blockDim.x;
            const uint32_t tot = build_prefix(a.T, nullptr, S, sm);
            // IU draws per thread in flight: their slot/flag loads, then their
            // table reads, then the stores (the chain is latency-bound otherwise)
            constexpr int IU = GX_I_UNROLL;
            const uint32_t T_all = (uint32_t)total_threads;
            for (uint32_t x0 = blockIdx.x * blockDim.x + tid; x0 < tot; x0 += IU * T_all) {
                // per item only (batch, position) and the two loaded words stay
                // live; addresses are recomputed (64-bit address arrays spilled)
                uint32_t bb[IU], pp[IU], ds[IU], rk[IU];
#pragma unroll
                for (int j = 0; j < IU; ++j) {
                    const uint32_t x = x0 + j * T_all;
                    ds[j] = kResolved;
                    rk[j] = 1;
                    bb[j] = 0;
                    pp[j] = 0;
                    if (x < tot) {
                        bb[j] = prefix_batch(sm, S, x);
                        pp[j] = x - sm.px[bb[j]];
                        const uint64_t gd = (uint64_t)bb[j] * a.cap_draw + pp[j];
                        ds[j] = a.dslot[gd];
                        rk[j] = a.drank[gd];
                    }
                }
                uint32_t val[IU];
                if (last_layer) {
                    // a loser's drank holds kNewBit | the winner's draw position
                    // (phase F), and the winner's drank its local id (phase H):
                    // no table read
#pragma unroll
                    for (int j = 0; j < IU; ++j)
                        if (!(ds[j] & kResolved) && (rk[j] & kNewBit))
                            val[j] = a.drank[(uint64_t)bb[j] * a.cap_draw + (rk[j] & ~kNewBit)];
#pragma unroll
                    for (int j = 0; j < IU; ++j)
                        if (!(ds[j] & kResolved) && (rk[j] & kNewBit))
                            a.edges[(uint64_t)bb[j] * a.cap_e_batch + a.e_off[l] + pp[j]].x = val[j];
                } else {
#pragma unroll
                    for (int j = 0; j < IU; ++j)  // resolved at insert time or a winner: nothing to do
                        if (!(ds[j] & kResolved) && !rk[j]) val[j] = (uint32_t)tab[(uint64_t)bb[j] * a.tab_cap + ds[j]];
#pragma unroll
                    for (int j = 0; j < IU; ++j)
                        if (!(ds[j] & kResolved) && !rk[j])
                            a.edges[(uint64_t)bb[j] * a.cap_e_batch + a.e_off[l] + pp[j]].x = val[j];
                }
            }
            for (uint32_t b = blockIdx.x * blockDim.x + tid; b < S; b += total_threads) {
                a.layer_count[(uint64_t)b * a.L + l] = a.T[b];
                a.dbase[b] += a.T[b];
                a.F[b] = a.n_ids[b];
            }
        }
        grid_sync(a.bar);
        TRACE_STAMP(a, l, 5);
    }

    // ---- leave the live table clean for the next call (coalesced bulk clear) ----
    clear_region(cur ? a.tab1 : a.tab0, a.tab_cap, H, S);
    if (a.trace && blockIdx.x == 0) {
        __syncthreads();
        if (threadIdx.x == 0) a.trace[127] = gtimer() - a.trace[0];
    }
}

// ---------------------------------------------------------------------------
// Cluster sampler: one thread-block cluster (CS CTAs on CS SMs) owns a batch at
// a time and walks the batches of the launch independently of the other
// clusters. All synchronisation is the hardware cluster barrier; per-CTA
// partial sums are exchanged through distributed shared memory; the batch's
// dedup table is the cluster's private region in global memory, and since only
// gridDim/CS batches are live at once their tables stay L2-resident. Same
// phases and bit-exact outputs as k_sample (sampler.hpp:69-117).
// ---------------------------------------------------------------------------
constexpr int SC_THREADS = 512;

struct ClSmem {
    uint32_t scan[34];
    uint32_t part[4];       // partials published to the cluster
    uint32_t bc[4];
    unsigned long long red[34];
};

// sum over ranks < r (and total) of part[idx] published by every CTA of the cluster
__device__ __forceinline__ void cluster_prefix(cg::cluster_group& cl, ClSmem& sm, int idx, uint32_t CS,
                                               uint32_t* before, uint32_t* total) {
    if (threadIdx.x == 0) {
        uint32_t b = 0, t = 0;
        for (uint32_t r = 0; r < CS; ++r) {
            const uint32_t* rp = cl.map_shared_rank(sm.part, r);
            const uint32_t v = rp[idx];
            if (r < cl.block_rank()) b += v;
            t += v;
        }
        sm.bc[0] = b;
        sm.bc[1] = t;
    }
    __syncthreads();
    *before = sm.bc[0];
    *total = sm.bc[1];
    __syncthreads();
}

template <int CS>
__global__ void __launch_bounds__(SC_THREADS) k_sample_cl(SampArgs a) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ ClSmem sm;
    const uint32_t rank = cl.block_rank();
    const uint32_t cid = blockIdx.x / CS, ncl = gridDim.x / CS;
    const uint32_t tid = threadIdx.x, T = blockDim.x;
    const uint32_t ct = rank * T + tid, CT = CS * T;
    unsigned long long* tabs[2] = {a.tab0 + (uint64_t)cid * a.tab_cap, a.tab1 + (uint64_t)cid * a.tab_cap};
    unsigned long long io_pages = 0, io_lists = 0, io_bytes = 0;

    for (uint32_t b = cid; b < a.S; b += ncl) {
        const uint64_t ibase = (uint64_t)b * a.cap_ids;
        const uint32_t ns = (uint32_t)(a.seed_off[b + 1] - a.seed_off[b]);
        const uint64_t seed = a.bseed[b];
        uint32_t F = ns;
        uint64_t dbase = 0;
        uint32_t H = 0;
        int cur = 0;
        for (uint32_t l = 0; l < a.L || l == 0; ++l) {
            // ---- table (re)build: H = nextpow2(2 * min(cap, F (1 + f_l))) ----
            const unsigned long long need0 = (unsigned long long)F * (1ull + (a.L ? a.fan[l] : 0));
            const unsigned long long need = need0 < a.cap_ids ? need0 : (unsigned long long)a.cap_ids;
            uint32_t newH = 1024;
            while (newH < 2 * need) newH <<= 1;
            if (newH > a.tab_cap) newH = (uint32_t)a.tab_cap;
            if (l == 0 || newH != H) {
                unsigned long long* told = tabs[cur];
                unsigned long long* tnew = l == 0 ? told : tabs[cur ^ 1];
                if (l > 0)
                    for (uint32_t x = ct; x < H; x += CT) told[x] = kEmptySlot;
                for (uint32_t k = ct; k < F; k += CT) {
                    uint32_t v;
                    if (l == 0) {
                        v = a.seeds[a.seed_off[b] + k];
                        a.ids[ibase + k] = v;
                    } else {
                        v = __ldcg(a.ids + ibase + k);
                    }
                    bool dup = false;
                    table_insert(tnew, newH, v, k, l == 0 ? &dup : nullptr);
                    if (dup) atomicOr(&a.io[3], 1ull);
                }
                if (l > 0) cur ^= 1;
                H = newH;
                cl.sync();
            }
            if (a.L == 0) break;
            unsigned long long* tab = tabs[cur];
            const uint32_t f = a.fan[l];
            uint2* bedge = a.edges + (uint64_t)b * a.cap_e_batch + a.e_off[l];
            uint32_t* bdslot = a.dslot + (uint64_t)b * a.cap_draw;
            uint32_t* bdrank = a.drank + (uint64_t)b * a.cap_draw;

            // ---- A: per parent deg/take (this CTA's contiguous chunk), IoStats ----
            const uint32_t pch = (F + CS - 1) / CS;
            const uint32_t k0 = min(F, rank * pch), k1 = min(F, k0 + pch);
            uint32_t csum = 0;
            for (uint32_t k = k0 + tid; k < k1; k += T) {
                const uint64_t gi = ibase + k;
                const uint32_t v = __ldcg(a.ids + gi);  // written by other CTAs of the cluster
                const uint64_t lo = a.indptr[v], hi = a.indptr[v + 1];
                const uint32_t deg = (uint32_t)(hi - lo);
                const uint32_t take = min(f, deg);
                a.plo[gi] = lo;
                a.pdeg[gi] = deg;
                a.pscan[gi] = take;
                csum += take;
                if (!a.ncbits || !((__ldg(a.ncbits + (v >> 5)) >> (v & 31)) & 1u)) {
                    io_lists += 1;
                    io_pages += pages_touched(8 * lo, 8 * hi);
                    io_bytes += 8ull * deg;
                }
            }
            csum = block_sum(csum, sm.scan);
            if (tid == 0) sm.part[0] = csum;
            cl.sync();
            uint32_t doff, Tb;
            cluster_prefix(cl, sm, 0, CS, &doff, &Tb);

            // ---- E: positions per parent, then one draw per thread ----------------
            for (uint32_t r0 = k0; r0 < k1; r0 += T * 4) {
                uint32_t take[4], s = 0;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t k = r0 + tid * 4 + j;
                    take[j] = k < k1 ? a.pscan[ibase + k] : 0;
                    s += take[j];
                }
                uint32_t tot;
                uint32_t off = doff + block_excl_scan(s, sm.scan, tot);
                const uint32_t d0 = doff;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (take[j]) {
                        const uint32_t k = r0 + tid * 4 + j;
                        draw_positions(take[j], seed, dbase + off, a.pdeg[ibase + k], bedge + off, k);
                    }
                    off += take[j];
                }
                __syncthreads();
                for (uint32_t p = d0 + tid; p < d0 + tot; p += T) {
                    const uint2 st = bedge[p];
                    const uint32_t child = ld_index(a, a.plo[ibase + st.y] + st.x);
                    bedge[p] = make_uint2(child, st.y);
                    bdslot[p] = table_insert(tab, H, child, kNewBit | p);
                }
                doff += tot;
                __syncthreads();
            }
            cl.sync();  // every insert of the layer is in the table

            // ---- F/H: first-occurrence winners ranked by draw position -------------
            const uint32_t dch = (Tb + CS - 1) / CS;
            const uint32_t p0 = min(Tb, rank * dch), p1 = min(Tb, p0 + dch);
            uint32_t wsum = 0;
            for (uint32_t p = p0 + tid; p < p1; p += T) {
                const uint32_t child = __ldcg(&bedge[p].x);
                const uint32_t fl =
                    __ldcg(tab + __ldcg(bdslot + p)) == (((unsigned long long)child << 32) | (kNewBit | p)) ? 1u : 0u;
                bdrank[p] = fl;
                wsum += fl;
            }
            wsum = block_sum(wsum, sm.scan);
            if (tid == 0) sm.part[1] = wsum;
            cl.sync();
            uint32_t wbefore, wtot;
            cluster_prefix(cl, sm, 1, CS, &wbefore, &wtot);
            uint32_t rk = wbefore;
            for (uint32_t q0 = p0; q0 < p1; q0 += T) {
                const uint32_t p = q0 + tid;
                const uint32_t fl = p < p1 ? bdrank[p] : 0;
                uint32_t tot;
                const uint32_t ex = block_excl_scan(fl, sm.scan, tot);
                if (fl) {
                    const uint32_t child = __ldcg(&bedge[p].x);
                    const uint32_t local = F + rk + ex;
                    a.ids[ibase + local] = child;
                    tab[__ldcg(bdslot + p)] = ((unsigned long long)child << 32) | local;
                }
                rk += tot;
            }
            cl.sync();
            // ---- I: edge sources -> local ids --------------------------------------
            for (uint32_t p = ct; p < Tb; p += CT) bedge[p].x = (uint32_t)__ldcg(tab + __ldcg(bdslot + p));
            if (ct == 0) a.layer_count[(uint64_t)b * a.L + l] = Tb;
            dbase += Tb;
            F += wtot;
            cl.sync();
        }
        // leave this cluster's table clean for its next batch
        unsigned long long* tab = tabs[cur];
        for (uint32_t x = ct; x < H; x += CT) tab[x] = kEmptySlot;
        if (ct == 0) a.n_ids[b] = F;
        cl.sync();
    }
    io_pages = warp_sum(io_pages);
    io_lists = warp_sum(io_lists);
    io_bytes = warp_sum(io_bytes);
    if ((tid & 31) == 0 && io_lists) {
        atomicAdd(&a.io[0], io_pages);
        atomicAdd(&a.io[1], io_lists);
        atomicAdd(&a.io[2], io_bytes);
    }
}

static uint64_t sat_mul(uint64_t a, uint64_t b, uint64_t cap) {
    if (a == 0 || b == 0) return 0;
    if (a > cap / b) return cap;
    return std::min(cap, a * b);
}

bool sample_run(gx_graph* g, const uint64_t* seeds_flat, const uint64_t* batch_off, uint64_t S,
                const uint32_t* fanouts, uint32_t L, const uint64_t* batch_seeds, gx_samples* out,
                uint32_t* firstx, uint32_t fx_epoch) {
    gx_ctx* ctx = g->ctx;
    if (L > (uint32_t)kMaxLayers) fail(GX_INVALID_ARGUMENT, "at most 16 layers are supported");
    uint64_t ns_max = 0, ns_total = batch_off[S];
    for (uint64_t b = 0; b < S; ++b) ns_max = std::max(ns_max, batch_off[b + 1] - batch_off[b]);
    const uint64_t N = g->n;
    // capacities: ids per batch <= min(N, ns * prod(1+f)); edges per layer <= bound_F_l * f_l
    uint64_t cap_ids = ns_max;
    std::vector<uint64_t> boundF(L + 1);
    boundF[0] = ns_max;
    for (uint32_t l = 0; l < L; ++l)
        boundF[l + 1] = std::min(std::max(N, ns_max),
                                 boundF[l] + sat_mul(boundF[l], fanouts[l], 1ull << 40));
    cap_ids = std::max<uint64_t>(boundF[L], 1);
    cap_ids = (cap_ids + 3) & ~3ull;
    out->ctx = ctx;
    out->S = S;
    out->L = L;
    out->fanouts.assign(fanouts, fanouts + L);
    out->cap_ids = cap_ids;
    out->cap_e.assign(L, 0);
    out->e_off.assign(L, 0);
    uint64_t ce = 0, cap_draw = 1;
    for (uint32_t l = 0; l < L; ++l) {
        uint64_t c = sat_mul(std::min(boundF[l], cap_ids), fanouts[l], 1ull << 40);
        if (c >= (1ull << 31)) fail(GX_INVALID_ARGUMENT, "batch too large: > 2^31 draws per layer");
        out->e_off[l] = ce;
        out->cap_e[l] = c;
        ce += (c + 3) & ~3ull;  // (layer regions in multiples of 4 edges: 16-byte aligned, see GX_SB_VEC)
        cap_draw = std::max<uint64_t>(cap_draw, (c + 3) & ~3ull);
    }
    out->cap_e_batch = std::max<uint64_t>(ce, 1);
    out->ids.reserve(S * cap_ids);
    out->n_ids.reserve(S);
    out->edges.reserve(S * out->cap_e_batch);
    out->layer_count.reserve(std::max<uint64_t>(S * L, 1));

    // Scratch is sized for one launch of at most kChunk batches; larger
    // superbatches run as consecutive launches into the same output (batches
    // are independent, sampler.hpp:216).
    static const uint64_t chunk = [] {  // batches per launch (GX_SAMPLER_CHUNK)
        const char* e = std::getenv("GX_SAMPLER_CHUNK");
        const long v = e ? std::atol(e) : (long)kChunk;
        return (uint64_t)std::min<long>(std::max<long>(v, 1), (long)kMaxBatchesPerLaunch);
    }();
    const uint64_t CH = std::min<uint64_t>(S, chunk);
    SampleScratch& ss = ctx->ss;
    cudaStream_t st = ctx->stream;
    ss.F.reserve(CH);
    ss.T.reserve(CH);
    ss.dbase.reserve(CH);
    ss.bseed.reserve(S);
    ss.seed_off.reserve(S + 1);
    ss.seeds32.reserve(std::max<uint64_t>(ns_total, 1));
    ss.pscan.reserve(CH * cap_ids);
    ss.pdeg.reserve(CH * cap_ids);
    ss.plo.reserve(CH * cap_ids);
    ss.idslot.reserve(CH * cap_ids);
    const uint64_t max_tiles = CH * ((std::max(cap_ids, cap_draw) + SB_TILE - 1) / SB_TILE) + 1;
    ss.tsum.reserve(max_tiles);
    ss.tsum2.reserve(max_tiles);
    ss.dslot.reserve(CH * cap_draw);
    ss.drank.reserve(CH * cap_draw);
    uint64_t tab_cap = 1024;
    while (tab_cap < 2 * cap_ids) tab_cap <<= 1;
    if (tab_cap > (1ull << 31)) fail(GX_INVALID_ARGUMENT, "batch too large for the dedup table");
    if (CH * tab_cap > ss.tab_slots) {
        for (int i = 0; i < 2; ++i) {
            ss.tab[i].alloc(CH * tab_cap);
            GX_CUDA(cudaMemsetAsync(ss.tab[i].p, 0xff, ss.tab[i].bytes(), st));
        }
        ss.tab_slots = CH * tab_cap;
    }
    ss.io.reserve(4);
    ss.tctr.reserve(4 * kMaxLayers);
    GX_CUDA(cudaMemsetAsync(ss.io.p, 0, 4 * sizeof(unsigned long long), st));

    // host -> device: seeds (u32), offsets, batch seeds
    std::vector<uint32_t> s32(std::max<uint64_t>(ns_total, 1));
    for (uint64_t i = 0; i < ns_total; ++i) s32[i] = (uint32_t)seeds_flat[i];
    GX_CUDA(cudaMemcpyAsync(ss.seeds32.p, s32.data(), ns_total * 4, cudaMemcpyHostToDevice, st));
    GX_CUDA(cudaMemcpyAsync(ss.seed_off.p, batch_off, (S + 1) * 8, cudaMemcpyHostToDevice, st));
    GX_CUDA(cudaMemcpyAsync(ss.bseed.p, batch_seeds, S * 8, cudaMemcpyHostToDevice, st));

    SampArgs a{};
    a.indptr = g->indptr.p;
    a.indices = g->indices.p;
    if (g->part.P) {
        if (!g->part.attached) fail(GX_LOGIC_ERROR, "partitioned graph: peers are not attached");
        a.nparts = (uint32_t)g->part.P;
        for (int q = 0; q < g->part.P; ++q) a.part[q] = g->part.ptr[q];
        for (int q = 0; q <= g->part.P; ++q) a.ebound[q] = g->part.ebound[q];
    }
    a.N = N;
    a.L = L;
    for (uint32_t l = 0; l < L; ++l) {
        a.fan[l] = fanouts[l];
        a.e_off[l] = out->e_off[l];
    }
    a.seeds = ss.seeds32.p;
    a.cap_ids = cap_ids;
    a.cap_e_batch = out->cap_e_batch;
    a.F = ss.F.p;
    a.T = ss.T.p;
    a.dbase = ss.dbase.p;
    a.pscan = ss.pscan.p;
    a.plo = ss.plo.p;
    a.pdeg = ss.pdeg.p;
    a.idslot = ss.idslot.p;
    a.tsum = ss.tsum.p;
    a.tsum2 = ss.tsum2.p;
    a.dslot = ss.dslot.p;
    a.drank = ss.drank.p;
    a.cap_draw = cap_draw;
    a.tab0 = ss.tab[0].p;
    a.tab1 = ss.tab[1].p;
    a.tab_cap = tab_cap;
    a.io = ss.io.p;
    a.ncbits = g->ncache_bits;
    // first-use keys (b << 21 | local) need local ids below 2^21 and S <= 2048
    const bool fx_ok = firstx && cap_ids <= (1ull << 21) && S <= 2048;
    a.firstx = fx_ok ? firstx : nullptr;
    a.fx_epoch = fx_epoch;
    a.tctr = ss.tctr.p;
    a.bar = ctx->barrier.p;
    static const bool trace = std::getenv("GX_SAMPLER_TRACE") != nullptr;
    static DevBuf<unsigned long long> tbuf;
    if (trace) {
        tbuf.reserve(128);
        GX_CUDA(cudaMemsetAsync(tbuf.p, 0, 128 * 8, st));
        a.trace = tbuf.p;
    }

    // phase-E draw staging in shared memory when a tile's draws fit 32 KB
    // (SB_TILE parents x max fanout; GX_SAMPLER_STAGE_SMEM=0 keeps the edge slots)
    uint32_t maxf = 0;
    for (uint32_t l = 0; l < L; ++l) maxf = std::max(maxf, fanouts[l]);
    const size_t stage_bytes = (size_t)SB_TILE * maxf * sizeof(uint2);
    static const bool stage_knob = env_int("GX_SAMPLER_STAGE_SMEM", 1) != 0;
    a.stage_smem = stage_knob && maxf > 0 && stage_bytes <= (32u << 10) ? 1u : 0u;
    const size_t smem = ((sizeof(SampSmem) + 15) & ~size_t(15)) + (a.stage_smem ? stage_bytes : 0);
    // attributes and occupancy are per device (and per shared-memory size)
    static PerDevice<std::map<size_t, int>> bps_dev;
    GX_CUDA(cudaSetDevice(ctx->device));
    int blocks_per_sm = 0;
    {
        auto lk = bps_dev.lock();
        int& cached = bps_dev.at(ctx->device)[smem];
        // the attribute is per kernel: keep it at the largest size used on this device
        int& attr = bps_dev.at(ctx->device)[0];
        if ((int)smem > attr) {
            GX_CUDA(cudaFuncSetAttribute(k_sample, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr = (int)smem;
        }
        if (cached < 1) {
            static const int carve = env_int("GX_SAMPLER_CARVEOUT", -1);  // % of the array as shared memory
            if (carve >= 0)
                GX_CUDA(cudaFuncSetAttribute(k_sample, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
            GX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cached, k_sample, SB_THREADS, smem));
            if (cached < 1) fail(GX_CUDA_ERROR, "sampler kernel cannot be resident");
        }
        blocks_per_sm = cached;
    }
    // CTAs per SM (GX_SAMPLER_BPS, default GX_SB_MINB): all that fit
    static const int bps_use = [] {
        const char* e = std::getenv("GX_SAMPLER_BPS");
        return e ? std::max(1, std::atoi(e)) : GX_SB_MINB;
    }();
    static const int ctas_knob = env_int("GX_SAMPLER_CTAS", 0);  // explicit CTA count (0 = per-SM rule)
    const int ctas_max = ctx->num_sms * std::min(bps_use, blocks_per_sm);
    dim3 grid(ctas_knob > 0 ? std::min(ctas_knob, ctas_max) : ctas_max), block(SB_THREADS);
    // cluster sampler (GX_SAMPLER_CLUSTER = 8 or 16 CTAs per batch; 0 = grid-wide kernel)
    static const int cs = [] {
        const char* e = std::getenv("GX_SAMPLER_CLUSTER");
        const int v = e ? std::atoi(e) : 0;  // measured slower than the grid kernel at B=1000
        return (v == 8 || v == 16) ? v : 0;
    }();
    if (cs) {
        static PerDevice<bool> attr_dev;
        {
            auto lk = attr_dev.lock();
            bool& attr = attr_dev.at(ctx->device);
            if (!attr) {
                GX_CUDA(cudaFuncSetAttribute(k_sample_cl<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
                attr = true;
            }
        }
        const uint32_t ncl = std::max(1, ctx->num_sms / cs);
        for (uint64_t c0 = 0; c0 < S; c0 += CH) {
            const uint64_t nb = std::min(CH, S - c0);
            a.S = (uint32_t)nb;
            a.bseed = ss.bseed.p + c0;
            a.seed_off = ss.seed_off.p + c0;
            a.ids = out->ids.p + c0 * cap_ids;
            a.n_ids = out->n_ids.p + c0;
            a.edges = out->edges.p + c0 * out->cap_e_batch;
            a.layer_count = out->layer_count.p + c0 * L;
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3(ncl * cs);
            lc.blockDim = dim3(SC_THREADS);
            lc.dynamicSmemBytes = 0;
            lc.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            if (cs == 16) GX_CUDA(cudaLaunchKernelEx(&lc, k_sample_cl<16>, a));
            else GX_CUDA(cudaLaunchKernelEx(&lc, k_sample_cl<8>, a));
            GX_CHECK_LAUNCH();
        }
        return false;  // the cluster sampler does not fill the first-use array
    }
    for (uint64_t c0 = 0; c0 < S; c0 += CH) {
        const uint64_t nb = std::min(CH, S - c0);
        a.S = (uint32_t)nb;
        a.bseed = ss.bseed.p + c0;
        a.seed_off = ss.seed_off.p + c0;  // global offsets into the flat seed array
        a.ids = out->ids.p + c0 * cap_ids;
        a.n_ids = out->n_ids.p + c0;
        a.edges = out->edges.p + c0 * out->cap_e_batch;
        a.layer_count = out->layer_count.p + c0 * L;
        a.batch0 = (uint32_t)c0;
        void* args[] = {&a};
        barrier_reset(a.bar, st);
        if (coop_launch()) GX_CUDA(cudaLaunchCooperativeKernel((void*)k_sample, grid, block, args, smem, st));
        else GX_CUDA(cudaLaunchKernel((void*)k_sample, grid, block, args, smem, st));
        GX_CHECK_LAUNCH();
        if (trace) {
            unsigned long long h[128];
            GX_CUDA(cudaMemcpyAsync(h, tbuf.p, sizeof h, cudaMemcpyDeviceToHost, st));
            GX_CUDA(cudaStreamSynchronize(st));
            const char* names[6] = {"D", "A", "E", "F", "H", "I"};
            unsigned long long prev = 0;
            std::string line = "[sampler trace us]";
            for (uint32_t l = 0; l < std::max<uint32_t>(L, 1); ++l)
                for (int ph = 0; ph < 6; ++ph) {
                    const unsigned long long t = h[1 + l * 8 + ph];
                    if (!t) continue;
                    line += " L" + std::to_string(l) + names[ph] + "=" + std::to_string((t - prev) / 1000.0).substr(0, 6);
                    prev = t;
                }
            line += " end=" + std::to_string((h[127] - prev) / 1000.0).substr(0, 6);
            // E1/E2 split: cycles summed over CTAs / CTAs / SM clock (~1.9 GHz) = us per CTA
            for (uint32_t l = 0; l < std::min<uint32_t>(L, 8); ++l)
                line += " L" + std::to_string(l) + "E1/E2(us/CTA)=" +
                        std::to_string(h[100 + 2 * l] / (double)grid.x / 1965.0).substr(0, 6) + "/" +
                        std::to_string(h[101 + 2 * l] / (double)grid.x / 1965.0).substr(0, 6);
            fprintf(stderr, "%s\n", line.c_str());
        }
    }
    return fx_ok;
}

void samples_sync_host(gx_samples* s) {
    cudaStream_t st = s->ctx->stream;
    s->h_n_ids.resize(s->S);
    s->h_layer_count.resize(s->S * s->L);
    // one pinned landing area [io u64 x3 | n_ids S | layer_count S*L]: the
    // copies stay asynchronous and the host waits once
    const size_t nl = s->S * s->L;
    s->h_pin.reserve(8 + s->S + nl);
    uint32_t* hp = s->h_pin.p;
    GX_CUDA(cudaMemcpyAsync(hp, s->ctx->ss.io.p, 4 * 8, cudaMemcpyDeviceToHost, st));
    GX_CUDA(cudaMemcpyAsync(hp + 8, s->n_ids.p, s->S * 4, cudaMemcpyDeviceToHost, st));
    if (nl) GX_CUDA(cudaMemcpyAsync(hp + 8 + s->S, s->layer_count.p, nl * 4, cudaMemcpyDeviceToHost, st));
    GX_CUDA(cudaStreamSynchronize(st));
    unsigned long long io[4];
    std::memcpy(io, hp, sizeof(io));
    std::memcpy(s->h_n_ids.data(), hp + 8, s->S * 4);
    if (nl) std::memcpy(s->h_layer_count.data(), hp + 8 + s->S, nl * 4);
    s->dup_seed = io[3] != 0;
    s->io.pages_read = io[0];
    s->io.neighbor_lists_read = io[1];
    s->io.bytes_read = io[2];
    s->io.rows_read = 0;
}

// Host-side seed validation in the reference's order (sampler.hpp:72,80-85):
// empty -> invalid_argument; per seed in order: >= N -> out_of_range,
// already seen -> invalid_argument.
static void validate_seeds(const uint64_t* seeds, uint64_t n, uint64_t N) {
    if (n == 0) fail(GX_INVALID_ARGUMENT, "sample_batch: seeds are empty");
    std::unordered_set<uint64_t> seen;
    seen.reserve(n * 2);
    for (uint64_t i = 0; i < n; ++i) {
        if (seeds[i] >= N) fail(GX_OUT_OF_RANGE, "seed node out of range");
        if (!seen.insert(seeds[i]).second) fail(GX_INVALID_ARGUMENT, "duplicate seed in batch");
    }
}

}  // namespace gx

using namespace gx;

extern "C" {

gx_status gx_sample_superbatch(gx_graph* g, const uint64_t* seeds_flat, const uint64_t* batch_off,
                               uint64_t n_batches, const uint32_t* fanouts, uint32_t n_layers,
                               uint64_t global_seed, uint64_t first_global_batch, gx_samples** out,
                               gx_iostats* io) {
    return guard([&] {
        if (!g || !out) fail(GX_INVALID_ARGUMENT, "null handle");
        // superbatch_sample wraps any per-batch failure into runtime_error (sampler.hpp:236)
        for (uint64_t b = 0; b < n_batches; ++b) {
            try {
                validate_seeds(seeds_flat + batch_off[b], batch_off[b + 1] - batch_off[b], g->n);
            } catch (const Error& e) {
                fail(GX_RUNTIME_ERROR, "superbatch sample failed: " + e.msg);
            }
        }
        std::vector<uint64_t> bs(std::max<uint64_t>(n_batches, 1));
        for (uint64_t i = 0; i < n_batches; ++i) bs[i] = derive_seed(global_seed, first_global_batch + i);
        auto s = new gx_samples();
        try {
            s->h_n_seeds.resize(n_batches);
            for (uint64_t b = 0; b < n_batches; ++b) s->h_n_seeds[b] = batch_off[b + 1] - batch_off[b];
            if (n_batches) {
                sample_run(g, seeds_flat, batch_off, n_batches, fanouts, n_layers, bs.data(), s);
                samples_sync_host(s);
            } else {
                s->ctx = g->ctx;
                s->L = n_layers;
                s->fanouts.assign(fanouts, fanouts + n_layers);
            }
        } catch (...) {
            delete s;
            throw;
        }
        if (io) {
            io->pages_read += s->io.pages_read;
            io->neighbor_lists_read += s->io.neighbor_lists_read;
            io->bytes_read += s->io.bytes_read;
        }
        *out = s;
    });
}

gx_status gx_sample_batch(gx_graph* g, const uint64_t* seeds, uint64_t n_seeds,
                          const uint32_t* fanouts, uint32_t n_layers, uint64_t batch_seed,
                          gx_samples** out, gx_iostats* io) {
    return guard([&] {
        if (!g || !out) fail(GX_INVALID_ARGUMENT, "null handle");
        validate_seeds(seeds, n_seeds, g->n);
        uint64_t off[2] = {0, n_seeds};
        auto s = new gx_samples();
        try {
            s->h_n_seeds.assign(1, n_seeds);
            sample_run(g, seeds, off, 1, fanouts, n_layers, &batch_seed, s);
            samples_sync_host(s);
        } catch (...) {
            delete s;
            throw;
        }
        if (io) {
            io->pages_read += s->io.pages_read;
            io->neighbor_lists_read += s->io.neighbor_lists_read;
            io->bytes_read += s->io.bytes_read;
        }
        *out = s;
    });
}

void gx_samples_destroy(gx_samples* s) { delete s; }
uint64_t gx_samples_num_batches(const gx_samples* s) { return s ? s->S : 0; }
uint32_t gx_samples_num_layers(const gx_samples* s) { return s ? s->L : 0; }

gx_status gx_samples_batch_info(const gx_samples* s, uint64_t b, uint64_t* n_ids, uint64_t* n_seeds,
                                uint64_t* layer_counts) {
    return guard([&] {
        if (!s || b >= s->S) fail(GX_OUT_OF_RANGE, "batch index out of range");
        if (n_ids) *n_ids = s->h_n_ids[b];
        if (n_seeds) *n_seeds = s->h_n_seeds[b];
        if (layer_counts)
            for (uint32_t l = 0; l < s->L; ++l) layer_counts[l] = s->h_layer_count[b * s->L + l];
    });
}

gx_status gx_samples_copy_ids(const gx_samples* s, uint64_t b, uint64_t* ids) {
    return guard([&] {
        if (!s || b >= s->S) fail(GX_OUT_OF_RANGE, "batch index out of range");
        const uint64_t n = s->h_n_ids[b];
        std::vector<uint32_t> tmp(n);
        GX_CUDA(cudaMemcpy(tmp.data(), s->ids.p + b * s->cap_ids, n * 4, cudaMemcpyDeviceToHost));
        for (uint64_t i = 0; i < n; ++i) ids[i] = tmp[i];
    });
}

gx_status gx_samples_copy_edges(const gx_samples* s, uint64_t b, uint32_t layer, uint32_t* pairs) {
    return guard([&] {
        if (!s || b >= s->S) fail(GX_OUT_OF_RANGE, "batch index out of range");
        if (layer >= s->L) fail(GX_OUT_OF_RANGE, "layer index out of range");
        const uint64_t n = s->h_layer_count[b * s->L + layer];
        GX_CUDA(cudaMemcpy(pairs, s->edges.p + b * s->cap_e_batch + s->e_off[layer], n * 8,
                           cudaMemcpyDeviceToHost));
    });
}

uint64_t gx_samples_total_edges(const gx_samples* s) {
    uint64_t t = 0;
    if (s)
        for (auto c : s->h_layer_count) t += c;
    return t;
}

}  // extern "C"
