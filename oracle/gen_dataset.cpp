// oracle/gen_dataset.cpp -- TEST INFRASTRUCTURE (never the product).
//
// A multi-threaded restatement of the reference's dataset synthesis that
// writes graph.bin / features.bin byte-identical to generate_dataset
// (graphgen.hpp:32-108, graph_store.hpp:53-98 + 237-262), so that the
// reference arm of bench.py can build papers100M-shape inputs on the host
// cores without the CUDA library (the reference's own single-threaded
// generator would need ~52 GB of pair vectors and tens of minutes at 1.6B
// edges). Pinned against the compiled reference generator in
// tests/test_oracle.py::test_threaded_generator_matches_reference.
//
//  * R-MAT attempt t consumes draws [t*scale, (t+1)*scale) of one SplitMix64
//    stream (graphgen.hpp:32-50); draw j = mix64(seed + j*gamma)
//    (common.hpp:72-77, 90-95), so attempts are generated in parallel blocks
//    and the accepted ones kept in attempt order until floor(n*avg_degree)
//    are accepted (graphgen.hpp:55-70).
//  * build_csc (graph_store.hpp:53-81): edges bucketed by destination,
//    each bucket sorted by (dst, src) and deduplicated; the in-neighbour
//    lists come out sorted, exactly as the per-node std::sort + std::unique.
//  * persist_graph (graph_store.hpp:83-98) and FeatureWriter
//    (graph_store.hpp:237-262) layouts; feature_value (graphgen.hpp:74-77).
#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cstdint>
#include <cstring>
#include <fcntl.h>
#include <string>
#include <sys/mman.h>
#include <thread>
#include <unistd.h>
#include <vector>

namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kPage = 4096;

inline uint64_t mix64(uint64_t z) {
    z += kGamma;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

inline float feature_value(uint64_t seed, uint64_t node, uint32_t col) {
    uint64_t h = mix64(seed ^ mix64(node * 0x10001ULL + col));
    return static_cast<float>(h >> 40) * 0x1.0p-24f;
}

template <class F>
void parallel(int threads, F&& f) {
    std::vector<std::thread> ts;
    for (int t = 0; t < threads; ++t) ts.emplace_back(f, t);
    for (auto& t : ts) t.join();
}

struct Map {
    int fd = -1;
    uint8_t* p = nullptr;
    uint64_t size = 0;
    int open(const char* path, uint64_t sz) {
        fd = ::open(path, O_RDWR | O_CREAT | O_TRUNC, 0644);
        if (fd < 0) return -1;
        if (ftruncate(fd, (off_t)sz) != 0) return -1;
        size = sz;
        void* m = mmap(nullptr, sz, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        if (m == MAP_FAILED) return -1;
        p = static_cast<uint8_t*>(m);
        return 0;
    }
    ~Map() {
        if (p) munmap(p, size);
        if (fd >= 0) ::close(fd);
    }
};

inline void put_u32(uint8_t* p, uint32_t v) { memcpy(p, &v, 4); }  // little-endian host (x86-64)
inline void put_u64(uint8_t* p, uint64_t v) { memcpy(p, &v, 8); }

}  // namespace

extern "C" {

// 0 ok, 1 invalid argument, 4 runtime (I/O) error
int gxg_graph_file(const char* path, uint64_t n, double avg_deg, double a, double b, double c,
                   uint64_t seed, int threads, uint64_t* n_edges) {
    if (n < 1 || avg_deg < 0 || n > (1ULL << 32) || threads < 1) return 1;
    unsigned scale = 0;
    while ((1ULL << scale) < n) ++scale;
    const uint64_t target = static_cast<uint64_t>(avg_deg * static_cast<double>(n));
    const double ab = a + b, abc = a + b + c;
    // accepted edges as (dst << 32 | src), in attempt order
    std::vector<uint64_t> keys(target ? target : 1);
    const uint64_t chunk = 1 << 22;  // attempts per thread per round
    std::vector<std::vector<uint64_t>> local(threads);
    uint64_t have = 0, attempt0 = 0;
    while (have < target) {
        parallel(threads, [&](int t) {
            auto& out = local[t];
            out.clear();
            const uint64_t a0 = attempt0 + (uint64_t)t * chunk;
            for (uint64_t at = a0; at < a0 + chunk; ++at) {
                uint64_t s = 0, d = 0;
                uint64_t ctr = seed + at * scale * kGamma;
                for (unsigned lv = 0; lv < scale; ++lv, ctr += kGamma) {
                    const double x = static_cast<double>(mix64(ctr) >> 11) * 0x1.0p-53;
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
                out.push_back(d << 32 | s);
            }
        });
        for (int t = 0; t < threads && have < target; ++t) {
            const uint64_t k = std::min<uint64_t>(local[t].size(), target - have);
            memcpy(keys.data() + have, local[t].data(), k * 8);
            have += k;
        }
        attempt0 += (uint64_t)threads * chunk;
    }
    local.clear();
    local.shrink_to_fit();

    // bucket by destination high bits, then sort + unique per bucket
    const unsigned bbits = std::min<unsigned>(scale, 16);
    const unsigned shift = scale - bbits;
    const uint64_t B = 1ULL << bbits;
    const uint64_t m = target;
    std::vector<uint64_t> hist((uint64_t)threads * B, 0);
    auto range = [&](int t, uint64_t total, uint64_t& lo, uint64_t& hi) {
        lo = total * t / threads;
        hi = total * (t + 1) / threads;
    };
    parallel(threads, [&](int t) {
        uint64_t lo, hi;
        range(t, m, lo, hi);
        uint64_t* h = hist.data() + (uint64_t)t * B;
        for (uint64_t i = lo; i < hi; ++i) h[(keys[i] >> 32) >> shift]++;
    });
    std::vector<uint64_t> boff(B + 1, 0);
    {
        uint64_t run = 0;
        for (uint64_t k = 0; k < B; ++k) {
            boff[k] = run;
            for (int t = 0; t < threads; ++t) {
                const uint64_t c0 = hist[(uint64_t)t * B + k];
                hist[(uint64_t)t * B + k] = run;
                run += c0;
            }
        }
        boff[B] = run;
    }
    std::vector<uint64_t> tmp(m ? m : 1);
    parallel(threads, [&](int t) {
        uint64_t lo, hi;
        range(t, m, lo, hi);
        uint64_t* h = hist.data() + (uint64_t)t * B;
        for (uint64_t i = lo; i < hi; ++i) tmp[h[(keys[i] >> 32) >> shift]++] = keys[i];
    });
    keys.clear();
    keys.shrink_to_fit();
    std::vector<uint64_t> uniq(B + 1, 0);
    std::atomic<uint64_t> next{0};
    parallel(threads, [&](int) {
        for (uint64_t k; (k = next.fetch_add(1)) < B;) {
            uint64_t* s = tmp.data() + boff[k];
            uint64_t* e = tmp.data() + boff[k + 1];
            std::sort(s, e);
            uniq[k] = static_cast<uint64_t>(std::unique(s, e) - s);
        }
    });
    std::vector<uint64_t> uoff(B + 1, 0);
    for (uint64_t k = 0; k < B; ++k) uoff[k + 1] = uoff[k] + uniq[k];
    const uint64_t E = uoff[B];

    const uint64_t header = 8 + 4 + 8 + 8 + 8;
    const uint64_t ind_off = (header + (n + 1) * 8 + kPage - 1) / kPage * kPage;
    Map f;
    if (f.open(path, ind_off + E * 8) != 0) return 4;
    memcpy(f.p, "GXGRAPH1", 8);
    put_u32(f.p + 8, 1);
    put_u64(f.p + 12, n);
    put_u64(f.p + 20, E);
    put_u64(f.p + 28, ind_off);
    uint8_t* ip = f.p + header;           // indptr u64[n+1] (unaligned: header is 36 bytes)
    uint8_t* ind = f.p + ind_off;         // indices u64[E]
    // per-destination counts: destinations of one bucket never appear in another
    std::vector<uint64_t> cnt(n + 1, 0);
    next = 0;
    parallel(threads, [&](int) {
        for (uint64_t k; (k = next.fetch_add(1)) < B;) {
            const uint64_t* s = tmp.data() + boff[k];
            uint64_t o = uoff[k];
            for (uint64_t j = 0; j < uniq[k]; ++j, ++o) {
                put_u64(ind + 8 * o, s[j] & 0xFFFFFFFFULL);
                cnt[(s[j] >> 32) + 1]++;
            }
        }
    });
    {
        uint64_t run = 0;
        for (uint64_t v = 0; v <= n; ++v) {
            run += cnt[v];
            put_u64(ip + 8 * v, run);
        }
    }
    *n_edges = E;
    return 0;
}

int gxg_features_file(const char* path, uint64_t n, uint32_t dim, uint64_t value_seed, int threads) {
    if (n < 1 || dim < 1 || threads < 1) return 1;
    const uint64_t payload = kPage;  // header (36 bytes) padded to one page
    Map f;
    if (f.open(path, payload + n * dim * 4ULL) != 0) return 4;
    memcpy(f.p, "GXFEAT01", 8);
    put_u32(f.p + 8, 1);
    put_u64(f.p + 12, n);
    put_u32(f.p + 20, dim);
    put_u32(f.p + 24, 4);
    put_u64(f.p + 28, payload);
    float* rows = reinterpret_cast<float*>(f.p + payload);
    std::atomic<uint64_t> next{0};
    const uint64_t blk = 1 << 14;
    parallel(threads, [&](int) {
        for (uint64_t b; (b = next.fetch_add(blk)) < n;) {
            const uint64_t e = std::min(n, b + blk);
            for (uint64_t v = b; v < e; ++v)
                for (uint32_t j = 0; j < dim; ++j) rows[v * dim + j] = feature_value(value_seed, v, j);
        }
    });
    return 0;
}

}  // extern "C"
