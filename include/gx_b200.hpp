// gx_b200.hpp -- header-only C++ adapter over the C-ABI (gx_b200.h) that
// re-exposes the reference's hot-path signatures (Ginex "gx",
// /root/reference/proj/include/gx) in namespace gx_b200, so a caller of
//   gx::sample_batch / superbatch_sample (sampler.hpp:69,197)
//   gx::build_access_index / compute_init_set / simulate_changesets /
//       precompute_changesets (changeset.hpp:124,137,228,468)
//   gx::FeatureCache ctor / gather / apply_changeset (feature_cache.hpp:19,58,89)
// switches by changing the namespace. gx_status is rethrown as the same C++
// exception type the reference throws at that point.
//
// Link: -I<repo>/include <repo>/paper_2208_09151_b200/libgx_b200.so
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iterator>
#include <filesystem>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "gx_b200.h"

namespace gx_b200 {

using NodeId = std::uint64_t;
using Fanouts = std::vector<std::uint32_t>;
using LocalEdge = std::pair<std::uint32_t, std::uint32_t>;

struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(gx_status s) {
    if (s == GX_OK) return;
    const std::string m = gx_last_error();
    switch (s) {
        case GX_INVALID_ARGUMENT: throw std::invalid_argument(m);
        case GX_OUT_OF_RANGE: throw std::out_of_range(m);
        case GX_LOGIC_ERROR: throw std::logic_error(m);
        case GX_OVERFLOW: throw std::overflow_error(m);
        case GX_CUDA_ERROR: throw cuda_error(m);
        default: throw std::runtime_error(m);
    }
}

// One device context per process (device from $GX_DEVICE, default 0).
inline gx_ctx* context() {
    static std::unique_ptr<gx_ctx, void (*)(gx_ctx*)> c(
        [] {
            gx_ctx* p = nullptr;
            const char* d = std::getenv("GX_DEVICE");
            check(gx_ctx_create(d ? std::atoi(d) : 0, &p));
            return p;
        }(),
        gx_ctx_destroy);
    return c.get();
}

// common.hpp:32-45
struct IoStats {
    std::uint64_t pages_read = 0, rows_read = 0, neighbor_lists_read = 0, bytes_read = 0;
    IoStats& operator+=(const IoStats& o) {
        pages_read += o.pages_read;
        rows_read += o.rows_read;
        neighbor_lists_read += o.neighbor_lists_read;
        bytes_read += o.bytes_read;
        return *this;
    }
    void add(const gx_iostats& c) {
        pages_read += c.pages_read;
        rows_read += c.rows_read;
        neighbor_lists_read += c.neighbor_lists_read;
        bytes_read += c.bytes_read;
    }
};

inline std::uint64_t mix64(std::uint64_t z) { return gx_mix64(z); }
inline std::uint64_t derive_seed(std::uint64_t b, std::uint64_t i) { return gx_derive_seed(b, i); }
inline std::uint64_t pages_touched(std::uint64_t lo, std::uint64_t hi) { return gx_pages_touched(lo, hi); }
inline std::uint64_t page_count_for_row(std::uint64_t w, std::uint64_t r) {
    std::uint64_t p = 0;
    check(gx_page_count_for_row(w, r, &p));
    return p;
}

// graph_store.hpp:106-197 (CSC resident in HBM)
class GraphFile {
public:
    static GraphFile open(const std::filesystem::path& path) {
        gx_graph* g = nullptr;
        check(gx_graph_open(context(), path.string().c_str(), &g));
        return GraphFile(g);
    }
    std::uint64_t num_nodes() const { return gx_graph_num_nodes(g_.get()); }
    std::uint64_t num_edges() const { return gx_graph_num_edges(g_.get()); }
    std::uint64_t in_degree(NodeId v) const {
        std::uint64_t d = 0;
        check(gx_graph_in_degree(g_.get(), v, &d));
        return d;
    }
    gx_graph* handle() const { return g_.get(); }

private:
    explicit GraphFile(gx_graph* g) : g_(g, gx_graph_destroy) {}
    std::shared_ptr<gx_graph> g_;
};

// sampler.hpp:36-40
struct SampleOutput {
    std::vector<NodeId> ids;
    std::size_t num_seeds = 0;
    std::vector<std::vector<LocalEdge>> layers;
};

// neighbor_cache.hpp: the static neighbor cache. The CSC is HBM-resident, so
// it changes only the sampler's IoStats (a cached list charges nothing).
class NeighborCache {
public:
    std::uint64_t cached_node_count() const { return gx_ncache_cached_nodes(c_.get()); }
    std::uint64_t bytes_used() const { return gx_ncache_bytes_used(c_.get()); }
    gx_ncache* handle() const { return c_.get(); }
    explicit NeighborCache(gx_ncache* c) : c_(c, gx_ncache_destroy) {}

private:
    std::shared_ptr<gx_ncache> c_;
};
// build_neighbor_cache / load_neighbor_cache / persist_neighbor_cache (neighbor_cache.hpp:88-148)
inline NeighborCache build_neighbor_cache(const GraphFile& graph, std::uint64_t budget_bytes,
                                          IoStats* stats = nullptr) {
    gx_ncache* c = nullptr;
    gx_iostats io{};
    check(gx_ncache_build(graph.handle(), budget_bytes, &io, &c));
    if (stats) stats->add(io);
    return NeighborCache(c);
}
inline NeighborCache load_neighbor_cache(const GraphFile& graph, const std::filesystem::path& path,
                                         IoStats* stats = nullptr) {
    gx_ncache* c = nullptr;
    gx_iostats io{};
    check(gx_ncache_open(graph.handle(), path.string().c_str(), &io, &c));
    if (stats) stats->add(io);
    return NeighborCache(c);
}
inline void persist_neighbor_cache(const NeighborCache& cache, const std::filesystem::path& path) {
    check(gx_ncache_write(cache.handle(), path.string().c_str()));
}
namespace detail {
struct UseNcache {  // installs the cache on the graph for one sampler call
    gx_graph* g;
    UseNcache(gx_graph* graph, const NeighborCache* c) : g(graph) {
        check(gx_graph_set_neighbor_cache(g, c ? c->handle() : nullptr));
    }
    ~UseNcache() { gx_graph_set_neighbor_cache(g, nullptr); }
};
}  // namespace detail

namespace detail {
inline SampleOutput batch_of(gx_samples* s, std::uint64_t b) {
    const std::uint32_t L = gx_samples_num_layers(s);
    std::uint64_t n_ids = 0, n_seeds = 0;
    std::vector<std::uint64_t> lc(L ? L : 1);
    check(gx_samples_batch_info(s, b, &n_ids, &n_seeds, lc.data()));
    SampleOutput o;
    o.ids.resize(n_ids);
    o.num_seeds = n_seeds;
    check(gx_samples_copy_ids(s, b, o.ids.data()));
    o.layers.resize(L);
    for (std::uint32_t l = 0; l < L; ++l) {
        std::vector<std::uint32_t> pairs(2 * lc[l]);
        check(gx_samples_copy_edges(s, b, l, pairs.data()));
        o.layers[l].resize(lc[l]);
        for (std::uint64_t k = 0; k < lc[l]; ++k) o.layers[l][k] = {pairs[2 * k], pairs[2 * k + 1]};
    }
    return o;
}
}  // namespace detail

// sample_batch (sampler.hpp:69-117)
inline SampleOutput sample_batch(const GraphFile& graph, const NeighborCache* cache,
                                 std::span<const NodeId> seeds, const Fanouts& fanouts,
                                 std::uint64_t batch_seed, IoStats& stats) {
    detail::UseNcache use(graph.handle(), cache);
    gx_samples* s = nullptr;
    gx_iostats io{};
    check(gx_sample_batch(graph.handle(), seeds.data(), seeds.size(), fanouts.data(),
                          (std::uint32_t)fanouts.size(), batch_seed, &s, &io));
    std::unique_ptr<gx_samples, void (*)(gx_samples*)> h(s, gx_samples_destroy);
    stats.add(io);
    return detail::batch_of(s, 0);
}

// sampler.hpp:188-192
struct SuperbatchSampleResult {
    IoStats io;
    std::uint64_t files_written = 0;
    std::uint64_t batches = 0;
};

// superbatch_sample (sampler.hpp:197-243); `workers` kept for signature parity
inline SuperbatchSampleResult superbatch_sample(const GraphFile& graph, const NeighborCache* cache,
                                                std::span<const std::vector<NodeId>> batch_slice,
                                                const Fanouts& fanouts, std::uint64_t global_seed,
                                                std::uint64_t first_global_batch, std::uint64_t sb_index,
                                                const std::filesystem::path& out_dir, unsigned workers) {
    (void)workers;
    detail::UseNcache use(graph.handle(), cache);
    std::filesystem::create_directories(out_dir);
    std::vector<NodeId> flat;
    std::vector<std::uint64_t> off{0};
    for (auto& b : batch_slice) {
        flat.insert(flat.end(), b.begin(), b.end());
        off.push_back(flat.size());
    }
    gx_samples* s = nullptr;
    gx_iostats io{};
    check(gx_sample_superbatch(graph.handle(), flat.data(), off.data(), batch_slice.size(), fanouts.data(),
                               (std::uint32_t)fanouts.size(), global_seed, first_global_batch, &s, &io));
    std::unique_ptr<gx_samples, void (*)(gx_samples*)> h(s, gx_samples_destroy);
    check(gx_samples_write_files(s, out_dir.string().c_str(), sb_index));
    SuperbatchSampleResult r;
    r.io.add(io);
    r.batches = batch_slice.size();
    r.files_written = 2 * r.batches;
    return r;
}

// changeset.hpp:161-178
struct Changeset {
    std::vector<NodeId> in_ids, out_ids;
    std::vector<std::uint64_t> in_positions;
    bool operator==(const Changeset&) const = default;
};
struct SimulationResult {
    std::vector<std::uint64_t> misses;
    std::uint64_t total_accesses = 0;
    std::uint64_t total_misses() const {
        std::uint64_t t = 0;
        for (auto m : misses) t += m;
        return t;
    }
};
struct AccessIndex {  // changeset.hpp:61-71
    std::vector<std::uint64_t> iters, ptr;
    std::uint64_t total_accesses() const { return iters.size() - 1; }
};

namespace detail {
template <class Trace>
void flatten(const Trace& t, std::vector<NodeId>& flat, std::vector<std::uint64_t>& off) {
    off.assign(1, 0);
    for (std::size_t i = 0; i < t.iterations(); ++i) {
        auto ids = t.ids(i);
        flat.insert(flat.end(), ids.begin(), ids.end());
        off.push_back(flat.size());
    }
}
inline Changeset iter_of(gx_changesets* cs, std::uint64_t i) {
    std::uint64_t ni = 0, no = 0, m = 0;
    check(gx_changesets_iter_info(cs, i, &ni, &no, &m));
    Changeset c;
    c.in_ids.resize(ni);
    c.in_positions.resize(ni);
    c.out_ids.resize(no);
    check(gx_changesets_copy_iter(cs, i, c.in_ids.data(), c.out_ids.data(), c.in_positions.data()));
    return c;
}
}  // namespace detail

// build_access_index (changeset.hpp:124-129)
template <class Trace>
AccessIndex build_access_index(const Trace& trace, std::uint64_t num_nodes) {
    std::vector<NodeId> flat;
    std::vector<std::uint64_t> off;
    detail::flatten(trace, flat, off);
    AccessIndex ix;
    ix.iters.resize(flat.size() + 1);
    ix.ptr.resize(num_nodes);
    check(gx_access_index(context(), flat.data(), off.data(), off.size() - 1, num_nodes, ix.iters.data(),
                          ix.ptr.data()));
    return ix;
}

// compute_init_set (changeset.hpp:137-153)
template <class Trace>
std::vector<NodeId> compute_init_set(const Trace& trace, std::uint64_t num_entries, std::uint64_t num_nodes) {
    if (num_entries == 0) return {};
    std::vector<NodeId> flat;
    std::vector<std::uint64_t> off;
    detail::flatten(trace, flat, off);
    gx_changesets* cs = nullptr;
    check(gx_precompute_trace(context(), flat.data(), off.data(), off.size() - 1, num_nodes, num_entries, &cs));
    std::unique_ptr<gx_changesets, void (*)(gx_changesets*)> h(cs, gx_changesets_destroy);
    std::vector<NodeId> init(gx_changesets_init_size(cs));
    std::uint64_t n = 0;
    check(gx_changesets_init(cs, init.data(), &n));
    return init;
}

// simulate_changesets (changeset.hpp:228-295). The device recomputes next use
// itself; `index` only supplies num_nodes (= ptr.size(), as in the reference).
template <class Trace, class Sink>
SimulationResult simulate_changesets(const AccessIndex& index, const Trace& trace, std::uint64_t num_entries,
                                     std::span<const NodeId> init, Sink&& sink) {
    std::vector<NodeId> flat;
    std::vector<std::uint64_t> off;
    detail::flatten(trace, flat, off);
    const std::uint64_t S = off.size() - 1;
    gx_changesets* cs = nullptr;
    check(gx_simulate_trace(context(), flat.data(), off.data(), S, index.ptr.size(), num_entries, init.data(),
                            init.size(), &cs));
    std::unique_ptr<gx_changesets, void (*)(gx_changesets*)> h(cs, gx_changesets_destroy);
    SimulationResult r;
    r.misses.resize(S);
    check(gx_changesets_misses(cs, r.misses.data()));
    r.total_accesses = flat.size();
    std::vector<NodeId> state(init.begin(), init.end());
    std::sort(state.begin(), state.end());
    for (std::uint64_t i = 0; i < S; ++i) {
        Changeset c = detail::iter_of(cs, i);
        std::vector<NodeId> out(c.out_ids), next;
        std::set_difference(state.begin(), state.end(), out.begin(), out.end(), std::back_inserter(next));
        std::vector<NodeId> in(c.in_ids);
        std::sort(in.begin(), in.end());
        state.clear();
        std::merge(next.begin(), next.end(), in.begin(), in.end(), std::back_inserter(state));
        sink(i, c, std::span<const NodeId>(state));
    }
    return r;
}

// precompute_changesets (changeset.hpp:468-484) over ids files
struct FileTrace {
    std::vector<std::filesystem::path> files;
    std::size_t iterations() const { return files.size(); }
    std::vector<NodeId> ids(std::size_t i) const {
        FILE* f = std::fopen(files[i].string().c_str(), "rb");
        if (!f) throw std::runtime_error("cannot open: " + files[i].string());
        char magic[8];
        std::uint64_t n = 0;
        if (std::fread(magic, 1, 8, f) != 8 || std::memcmp(magic, "GXIDS001", 8) != 0 ||
            std::fread(&n, 8, 1, f) != 1) {
            std::fclose(f);
            throw std::runtime_error("bad magic in " + files[i].string() + " (expected GXIDS001)");
        }
        std::vector<NodeId> v(n);
        if (n && std::fread(v.data(), 8, n, f) != n) {
            std::fclose(f);
            throw std::runtime_error("truncated file: " + files[i].string());
        }
        std::fclose(f);
        return v;
    }
};
struct PrecomputeResult {
    std::uint64_t files_written = 0;
    SimulationResult sim;
    std::uint64_t init_size = 0;
};
inline PrecomputeResult precompute_changesets(const FileTrace& trace, std::uint64_t num_nodes,
                                              std::uint64_t num_entries, const std::filesystem::path& out_dir,
                                              std::uint64_t sb_index) {
    std::vector<NodeId> flat;
    std::vector<std::uint64_t> off;
    detail::flatten(trace, flat, off);
    gx_changesets* cs = nullptr;
    check(gx_precompute_trace(context(), flat.data(), off.data(), off.size() - 1, num_nodes, num_entries, &cs));
    std::unique_ptr<gx_changesets, void (*)(gx_changesets*)> h(cs, gx_changesets_destroy);
    check(gx_changesets_write_files(cs, out_dir.string().c_str(), sb_index));
    PrecomputeResult r;
    r.files_written = trace.iterations() + 1;
    r.sim.misses.resize(off.size() - 1);
    check(gx_changesets_misses(cs, r.sim.misses.data()));
    r.sim.total_accesses = flat.size();
    r.init_size = gx_changesets_init_size(cs);
    return r;
}

// graph_store.hpp:222-234
struct RowMatrix {
    std::size_t rows = 0, dim = 0;
    std::vector<float> data;
    void resize(std::size_t r, std::size_t d) {
        rows = r;
        dim = d;
        data.resize(r * d);
    }
    std::span<float> row(std::size_t k) { return {data.data() + k * dim, dim}; }
    std::span<const float> row(std::size_t k) const { return {data.data() + k * dim, dim}; }
};

// graph_store.hpp:280-333. Default: payload loaded into HBM. GX_BACKING_FILE
// keeps the reference's storage model (rows stay in features.bin; misses are
// read with O_DIRECT page runs into pinned staging, the SSD tier);
// GX_BACKING_HOST keeps them in pinned host memory.
class FeatureFile {
public:
    static FeatureFile open(const std::filesystem::path& path, int backing = GX_BACKING_DEVICE) {
        gx_features* f = nullptr;
        check(gx_features_open(context(), path.string().c_str(), backing, &f));
        return FeatureFile(f);
    }
    std::uint64_t num_nodes() const { return gx_features_num_nodes(f_.get()); }
    std::uint32_t dim() const { return gx_features_dim(f_.get()); }
    std::uint64_t row_bytes() const { return gx_features_row_bytes(f_.get()); }
    gx_features* handle() const { return f_.get(); }

private:
    explicit FeatureFile(gx_features* f) : f_(f, gx_features_destroy) {}
    std::shared_ptr<gx_features> f_;
};

// feature_cache.hpp:15-138
class FeatureCache {
public:
    struct GatherCounts {
        std::uint64_t hits = 0, misses = 0;
    };
    FeatureCache(const FeatureFile& store, std::span<const NodeId> init_ids, std::uint64_t num_entries,
                 IoStats& stats)
        : dim_(store.dim()), c_(nullptr, gx_cache_destroy), b_(nullptr, gx_batch_destroy) {
        gx_cache* c = nullptr;
        gx_iostats io{};
        check(gx_cache_create(store.handle(), init_ids.data(), init_ids.size(), num_entries, &io, &c));
        c_.reset(c);
        stats.add(io);
        gx_batch* b = nullptr;
        check(gx_batch_create(context(), &b));
        b_.reset(b);
    }
    std::uint64_t num_entries() const { return gx_cache_num_entries(c_.get()); }
    std::uint32_t dim() const { return dim_; }
    bool contains(NodeId v) const {
        int r = 0;
        check(gx_cache_contains(c_.get(), v, &r));
        return r != 0;
    }
    std::vector<float> cached_row(NodeId v) const {
        std::vector<float> r(dim_);
        check(gx_cache_cached_row(c_.get(), v, r.data()));
        return r;
    }
    GatherCounts gather(const FeatureFile& store, std::span<const NodeId> ids, RowMatrix& out,
                        IoStats& stats) const {
        (void)store;
        GatherCounts cnt;
        gx_iostats io{};
        check(gx_cache_gather(c_.get(), ids.data(), ids.size(), b_.get(), &cnt.hits, &cnt.misses, &io));
        stats.add(io);
        out.resize(ids.size(), dim_);
        check(gx_batch_copy_to_host(b_.get(), out.data.data()));
        return cnt;
    }
    void apply_changeset(const RowMatrix& batch, std::span<const NodeId> ids, const Changeset& cs) {
        if (cs.in_ids.size() != cs.in_positions.size())
            throw std::invalid_argument("changeset arrays disagree in length");
        if (batch.rows != ids.size() || batch.dim != dim_)
            throw std::invalid_argument("batch buffer does not match ids");
        check(gx_batch_upload(b_.get(), batch.data.data(), batch.rows, (std::uint64_t)batch.dim * 4));
        check(gx_cache_apply(c_.get(), b_.get(), ids.data(), ids.size(), cs.in_ids.data(), cs.in_positions.data(),
                             cs.in_ids.size(), cs.out_ids.data(), cs.out_ids.size()));
    }
    std::vector<NodeId> resident_set() const {
        std::vector<NodeId> r(num_entries());
        std::uint64_t n = 0;
        check(gx_cache_resident_set(c_.get(), r.data(), r.size(), &n));
        r.resize(n);
        return r;
    }

private:
    std::uint32_t dim_;
    std::unique_ptr<gx_cache, void (*)(gx_cache*)> c_;
    std::unique_ptr<gx_batch, void (*)(gx_batch*)> b_;
};

}  // namespace gx_b200
