// oracle/ref_driver.cpp -- TEST INFRASTRUCTURE ONLY (never shipped, never measured
// as the product).
//
// A thin extern "C" shim over the UNMODIFIED reference headers under
// /root/reference/proj/include/gx (header-only C++20). It is compiled by
// oracle/Makefile straight from those headers into oracle/_ref/libgx_ref.so, so
// the tests can (a) pin the C restatement in oracle/gx_oracle.c against the real
// reference, (b) generate the golden fixtures in tests/golden/, and (c) serve as
// the `cpu_baseline` / `--impl reference` arm of bench.py.
//
// Nothing here re-implements reference logic: every entry point forwards to the
// reference function it names and only marshals plain arrays in and out.

#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>

#include "gx/baselines.hpp"
#include "gx/graphgen.hpp"
#include "gx/pipeline.hpp"

using namespace gx;

namespace {

thread_local std::string g_err;

// status codes mirror include/gx_b200.h (gx_status)
enum : int { OK = 0, INVALID_ARGUMENT = 1, OUT_OF_RANGE = 2, LOGIC_ERROR = 3, RUNTIME_ERROR = 4,
             OVERFLOW_ = 5 };

template <class F>
int guard(F&& f) {
    try {
        f();
        return OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return INVALID_ARGUMENT;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return OUT_OF_RANGE;
    } catch (const std::overflow_error& e) {
        g_err = e.what();
        return OVERFLOW_;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return LOGIC_ERROR;
    } catch (const std::exception& e) {
        g_err = e.what();
        return RUNTIME_ERROR;
    }
}

void put_io(const IoStats& s, uint64_t* io) {
    if (!io) return;
    io[0] = s.pages_read;
    io[1] = s.rows_read;
    io[2] = s.neighbor_lists_read;
    io[3] = s.bytes_read;
}

struct Graph {
    GraphFile g;
};
struct Feat {
    FeatureFile f;
};
struct Cache {
    std::unique_ptr<FeatureCache> c;
};

std::vector<std::vector<NodeId>> make_trace(const uint64_t* flat, const uint64_t* off, uint64_t S) {
    std::vector<std::vector<NodeId>> t(S);
    for (uint64_t i = 0; i < S; ++i) t[i].assign(flat + off[i], flat + off[i + 1]);
    return t;
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

} // namespace

extern "C" {

const char* gxr_last_error() { return g_err.c_str(); }

uint64_t gxr_mix64(uint64_t z) { return mix64(z); }
uint64_t gxr_derive_seed(uint64_t b, uint64_t i) { return derive_seed(b, i); }

// --- datasets --------------------------------------------------------------

int gxr_generate_dataset(const char* dir, uint64_t n, double avg_deg, uint32_t dim,
                         uint64_t edge_seed, uint64_t value_seed, uint64_t* num_edges) {
    return guard([&] {
        GenSpec s;
        s.num_nodes = n;
        s.avg_degree = avg_deg;
        s.dim = dim;
        s.edge_seed = edge_seed;
        s.value_seed = value_seed;
        auto r = generate_dataset(s, dir);
        if (num_edges) *num_edges = r.num_edges;
    });
}

/// generate_edges only (graphgen.hpp:55); fills src/dst up to cap.
int gxr_generate_edges(uint64_t n, double avg_deg, uint64_t edge_seed, uint64_t* src,
                       uint64_t* dst, uint64_t cap, uint64_t* count) {
    return guard([&] {
        GenSpec s;
        s.num_nodes = n;
        s.avg_degree = avg_deg;
        s.edge_seed = edge_seed;
        auto e = generate_edges(s);
        *count = e.size();
        for (uint64_t i = 0; i < e.size() && i < cap; ++i) {
            src[i] = e[i].first;
            dst[i] = e[i].second;
        }
    });
}

/// build_csc + persist_graph (graph_store.hpp:53,83) over an explicit edge list.
int gxr_write_graph(const char* path, uint64_t n, const uint64_t* src, const uint64_t* dst,
                    uint64_t m) {
    return guard([&] {
        std::vector<std::pair<NodeId, NodeId>> e(m);
        for (uint64_t i = 0; i < m; ++i) e[i] = {src[i], dst[i]};
        persist_graph(build_csc(e, n), path);
    });
}

/// persist_graph of a ready CSC (indptr n+1, indices e).
int gxr_write_graph_csc(const char* path, uint64_t n, const uint64_t* indptr,
                        const uint64_t* indices, uint64_t e) {
    return guard([&] {
        CscGraph g;
        g.num_nodes = n;
        g.indptr.assign(indptr, indptr + n + 1);
        g.indices.assign(indices, indices + e);
        persist_graph(g, path);
    });
}

float gxr_feature_value(uint64_t value_seed, uint64_t node, uint32_t col) {
    return feature_value(value_seed, node, col);
}

int gxr_write_features(const char* path, uint64_t n, uint32_t dim, const float* rows) {
    return guard([&] {
        FeatureWriter w(path, n, dim);
        for (uint64_t v = 0; v < n; ++v)
            w.append_row(std::span<const float>(rows + v * dim, dim));
        w.close();
    });
}

// --- graph handle ----------------------------------------------------------

int gxr_graph_open(const char* path, void** out) {
    return guard([&] { *out = new Graph{GraphFile::open(path)}; });
}
void gxr_graph_close(void* g) { delete static_cast<Graph*>(g); }
uint64_t gxr_graph_num_nodes(void* g) { return static_cast<Graph*>(g)->g.num_nodes(); }
uint64_t gxr_graph_num_edges(void* g) { return static_cast<Graph*>(g)->g.num_edges(); }
int gxr_graph_read_all(void* gh, uint64_t* indptr, uint64_t* indices) {
    return guard([&] {
        auto& g = static_cast<Graph*>(gh)->g;
        std::memcpy(indptr, g.indptr().data(), (g.num_nodes() + 1) * 8);
        IoStats s;
        std::vector<NodeId> list;
        for (NodeId v = 0; v < g.num_nodes(); ++v) {
            g.read_in_neighbors(v, list, s);
            std::memcpy(indices + g.indptr()[v], list.data(), list.size() * 8);
        }
    });
}

// --- sampler (sampler.hpp) -------------------------------------------------

/// sample_batch (sampler.hpp:69). edges_out holds (src,dst) u32 pairs, layer
/// after layer; layer_counts[l] gives each layer's edge count.
static int sample_batch_impl(void* gh, const NeighborCache* nc, const uint64_t* seeds, uint64_t n_seeds,
                             const uint32_t* fanouts, uint32_t n_layers, uint64_t batch_seed,
                             uint64_t* ids_out, uint64_t ids_cap, uint64_t* n_ids, uint32_t* edges_out,
                             uint64_t edges_cap, uint64_t* layer_counts, uint64_t* io) {
    return guard([&] {
        auto& g = static_cast<Graph*>(gh)->g;
        IoStats s;
        Fanouts f(fanouts, fanouts + n_layers);
        SampleOutput o = sample_batch(g, nc, std::span<const NodeId>(seeds, n_seeds), f,
                                      batch_seed, s);
        *n_ids = o.ids.size();
        if (o.ids.size() > ids_cap) throw std::runtime_error("ids_cap too small");
        std::memcpy(ids_out, o.ids.data(), o.ids.size() * 8);
        uint64_t k = 0;
        for (uint32_t l = 0; l < n_layers; ++l) {
            layer_counts[l] = o.layers[l].size();
            if (k + o.layers[l].size() > edges_cap) throw std::runtime_error("edges_cap too small");
            for (auto& [a, b] : o.layers[l]) {
                edges_out[2 * k] = a;
                edges_out[2 * k + 1] = b;
                ++k;
            }
        }
        put_io(s, io);
    });
}

int gxr_sample_batch(void* gh, const uint64_t* seeds, uint64_t n_seeds, const uint32_t* fanouts,
                     uint32_t n_layers, uint64_t batch_seed, uint64_t* ids_out, uint64_t ids_cap,
                     uint64_t* n_ids, uint32_t* edges_out, uint64_t edges_cap,
                     uint64_t* layer_counts, uint64_t* io) {
    return sample_batch_impl(gh, nullptr, seeds, n_seeds, fanouts, n_layers, batch_seed, ids_out, ids_cap,
                             n_ids, edges_out, edges_cap, layer_counts, io);
}

/// sample_batch with a static neighbor cache loaded from ncache.bin
/// (load_neighbor_cache, neighbor_cache.hpp:130-148; its own load is not charged).
int gxr_sample_batch_nc(void* gh, const char* ncache_path, const uint64_t* seeds, uint64_t n_seeds,
                        const uint32_t* fanouts, uint32_t n_layers, uint64_t batch_seed, uint64_t* ids_out,
                        uint64_t ids_cap, uint64_t* n_ids, uint32_t* edges_out, uint64_t edges_cap,
                        uint64_t* layer_counts, uint64_t* io) {
    NeighborCache nc;
    const int rc = guard([&] { nc = load_neighbor_cache(ncache_path); });
    if (rc) return rc;
    return sample_batch_impl(gh, &nc, seeds, n_seeds, fanouts, n_layers, batch_seed, ids_out, ids_cap, n_ids,
                             edges_out, edges_cap, layer_counts, io);
}

/// build_neighbor_cache (neighbor_cache.hpp:88-116) + persist_neighbor_cache.
int gxr_ncache_build(void* gh, uint64_t budget_bytes, const char* path, uint64_t* io, uint64_t* cached) {
    return guard([&] {
        auto& g = static_cast<Graph*>(gh)->g;
        IoStats s;
        NeighborCache c = build_neighbor_cache(g, budget_bytes, &s);
        persist_neighbor_cache(c, path);
        if (cached) *cached = c.cached_node_count();
        put_io(s, io);
    });
}

/// simulate_policy (baselines.hpp:64-143): policy 0 none, 1 static_degree
/// (out-degrees from the graph, compute_out_degrees), 2 lru, 3 belady.
int gxr_simulate_policy(void* gh, const uint64_t* flat, const uint64_t* off, uint64_t S, uint64_t K,
                        int policy, uint64_t* misses_out, uint64_t* total_accesses) {
    return guard([&] {
        auto& g = static_cast<Graph*>(gh)->g;
        struct T {
            const uint64_t* flat;
            const uint64_t* off;
            uint64_t S;
            std::size_t iterations() const { return S; }
            std::vector<NodeId> ids(std::size_t i) const {  // the Trace concept (changeset.hpp:44-55)
                return std::vector<NodeId>(flat + off[i], flat + off[i + 1]);
            }
        } tr{flat, off, S};
        const CachePolicy pol[4] = {CachePolicy::none, CachePolicy::static_degree, CachePolicy::lru,
                                    CachePolicy::belady};
        std::vector<std::uint64_t> outdeg;
        if (policy == 1) outdeg = g.compute_out_degrees();
        PolicyResult r = simulate_policy(tr, g.num_nodes(), K, pol[policy], outdeg);
        for (uint64_t i = 0; i < S; ++i) misses_out[i] = r.misses[i];
        *total_accesses = r.total_accesses;
    });
}

/// superbatch_sample (sampler.hpp:197) writing ids/adj runtime files.
int gxr_superbatch_sample(void* gh, const uint64_t* seeds_flat, const uint64_t* batch_off,
                          uint64_t n_batches, const uint32_t* fanouts, uint32_t n_layers,
                          uint64_t global_seed, uint64_t first_global_batch, uint64_t sb_index,
                          const char* out_dir, unsigned workers, uint64_t* io, double* seconds) {
    return guard([&] {
        auto& g = static_cast<Graph*>(gh)->g;
        std::vector<std::vector<NodeId>> batches(n_batches);
        for (uint64_t b = 0; b < n_batches; ++b)
            batches[b].assign(seeds_flat + batch_off[b], seeds_flat + batch_off[b + 1]);
        Fanouts f(fanouts, fanouts + n_layers);
        double t0 = now_s();
        auto r = superbatch_sample(g, nullptr, batches, f, global_seed, first_global_batch,
                                   sb_index, out_dir, workers);
        if (seconds) *seconds = now_s() - t0;
        put_io(r.io, io);
    });
}

int gxr_plan_seed_batches(const uint64_t* train, uint64_t n, uint64_t batch_size,
                          uint64_t epoch_seed, uint64_t* shuffled_out) {
    return guard([&] {
        SeedPlan p = plan_seed_batches(std::span<const NodeId>(train, n), batch_size, epoch_seed);
        uint64_t k = 0;
        for (auto& b : p.batches)
            for (auto v : b) shuffled_out[k++] = v;
    });
}

/// derive_train_ids (pipeline.hpp:384) via a real TrainingRunner on the given files.
int gxr_train_ids(const char* graph_path, const char* feature_path, uint64_t seed,
                  double train_fraction, uint64_t* out, uint64_t cap, uint64_t* n) {
    return guard([&] {
        RunConfig cfg;
        cfg.graph_path = graph_path;
        cfg.feature_path = feature_path;
        cfg.use_neighbor_cache = false;
        cfg.seed = seed;
        cfg.train_fraction = train_fraction;
        cfg.runtime_dir = std::filesystem::temp_directory_path() / "gxr_train_ids_rt";
        TrainingRunner tr(cfg);
        auto& t = tr.train_ids();
        *n = t.size();
        for (uint64_t i = 0; i < t.size() && i < cap; ++i) out[i] = t[i];
    });
}

// --- inspector (changeset.hpp) --------------------------------------------

/// build_access_index (changeset.hpp:124) over a memory trace.
int gxr_access_index(const uint64_t* flat, const uint64_t* off, uint64_t S, uint64_t N,
                     uint64_t* iters_out, uint64_t* ptr_out) {
    return guard([&] {
        auto t = make_trace(flat, off, S);
        AccessIndex ix = build_access_index(MemoryTrace{&t}, N);
        std::memcpy(iters_out, ix.iters.data(), ix.iters.size() * 8);
        std::memcpy(ptr_out, ix.ptr.data(), ix.ptr.size() * 8);
    });
}

int gxr_compute_init_set(const uint64_t* flat, const uint64_t* off, uint64_t S, uint64_t K,
                         uint64_t N, uint64_t* out, uint64_t* n) {
    return guard([&] {
        auto t = make_trace(flat, off, S);
        auto init = compute_init_set(MemoryTrace{&t}, K, N);
        *n = init.size();
        std::memcpy(out, init.data(), init.size() * 8);
    });
}

/// build_access_index + simulate_changesets (changeset.hpp:228) with an
/// explicit init set. Changesets are returned flat: in_ids/in_pos with
/// in_off[S+1], out_ids with out_off[S+1]. If use_naive, runs
/// naive_belady_oracle (changeset.hpp:301) instead.
int gxr_simulate(const uint64_t* flat, const uint64_t* off, uint64_t S, uint64_t N, uint64_t K,
                 const uint64_t* init, uint64_t n_init, int use_naive, uint64_t* misses,
                 uint64_t* in_ids, uint64_t* in_pos, uint64_t* in_off, uint64_t* out_ids,
                 uint64_t* out_off, uint64_t* state_out, uint64_t* state_off,
                 uint64_t state_cap, double* seconds) {
    return guard([&] {
        auto t = make_trace(flat, off, S);
        MemoryTrace mt{&t};
        uint64_t ki = 0, ko = 0, ks = 0;
        in_off[0] = 0;
        out_off[0] = 0;
        if (state_off) state_off[0] = 0;
        auto sink = [&](std::size_t i, const Changeset& cs, std::span<const NodeId> st) {
            for (std::size_t k = 0; k < cs.in_ids.size(); ++k) {
                in_ids[ki] = cs.in_ids[k];
                in_pos[ki] = cs.in_positions[k];
                ++ki;
            }
            for (auto v : cs.out_ids) out_ids[ko++] = v;
            in_off[i + 1] = ki;
            out_off[i + 1] = ko;
            if (state_out) {
                if (ks + st.size() > state_cap) throw std::runtime_error("state_cap too small");
                for (auto v : st) state_out[ks++] = v;
                state_off[i + 1] = ks;
            }
        };
        std::span<const NodeId> in(init, n_init);
        double t0 = now_s();
        SimulationResult r;
        if (use_naive) {
            r = naive_belady_oracle(mt, K, in, N, sink);
        } else {
            AccessIndex ix = build_access_index(mt, N);
            r = simulate_changesets(ix, mt, K, in, sink);
        }
        if (seconds) *seconds = now_s() - t0;
        for (uint64_t i = 0; i < S; ++i) misses[i] = r.misses[i];
    });
}

int gxr_dp_optimal_misses(const uint64_t* flat, const uint64_t* off, uint64_t S, uint64_t K,
                          uint64_t* out) {
    return guard([&] { *out = dp_optimal_misses(make_trace(flat, off, S), K); });
}

/// precompute_changesets (changeset.hpp:468) over ids files already in dir.
int gxr_precompute_changesets(const char* dir, uint64_t sb, uint64_t S, uint64_t N, uint64_t K,
                              uint64_t* misses, uint64_t* init_size, double* seconds) {
    return guard([&] {
        FileTrace tr;
        for (uint64_t i = 0; i < S; ++i) tr.files.push_back(ids_file_path(dir, sb, i));
        double t0 = now_s();
        auto r = precompute_changesets(tr, N, K, dir, sb);
        if (seconds) *seconds = now_s() - t0;
        if (misses)
            for (uint64_t i = 0; i < S; ++i) misses[i] = r.sim.misses[i];
        if (init_size) *init_size = r.init_size;
    });
}

// --- executor (feature_cache.hpp) -----------------------------------------

int gxr_features_open(const char* path, void** out) {
    return guard([&] { *out = new Feat{FeatureFile::open(path)}; });
}
void gxr_features_close(void* f) { delete static_cast<Feat*>(f); }
uint32_t gxr_features_dim(void* f) { return static_cast<Feat*>(f)->f.dim(); }

int gxr_cache_create(void* fh, const uint64_t* init, uint64_t n_init, uint64_t K, uint64_t* io,
                     void** out) {
    return guard([&] {
        IoStats s;
        auto c = new Cache{std::make_unique<FeatureCache>(static_cast<Feat*>(fh)->f,
                                                          std::span<const NodeId>(init, n_init),
                                                          K, s)};
        *out = c;
        put_io(s, io);
    });
}
void gxr_cache_destroy(void* c) { delete static_cast<Cache*>(c); }

int gxr_cache_gather(void* ch, void* fh, const uint64_t* ids, uint64_t n, float* out,
                     uint64_t* hits, uint64_t* misses, uint64_t* io) {
    return guard([&] {
        auto& c = *static_cast<Cache*>(ch)->c;
        auto& f = static_cast<Feat*>(fh)->f;
        RowMatrix m;
        IoStats s;
        auto cnt = c.gather(f, std::span<const NodeId>(ids, n), m, s);
        if (out && !m.data.empty()) std::memcpy(out, m.data.data(), m.data.size() * 4);
        *hits = cnt.hits;
        *misses = cnt.misses;
        put_io(s, io);
    });
}

int gxr_cache_apply(void* ch, const float* batch, uint64_t rows, uint32_t dim, const uint64_t* ids,
                    uint64_t n_ids, const uint64_t* in_ids, const uint64_t* in_pos, uint64_t n_in,
                    const uint64_t* out_ids, uint64_t n_out) {
    return guard([&] {
        auto& c = *static_cast<Cache*>(ch)->c;
        RowMatrix m;
        m.resize(rows, dim);
        if (rows) std::memcpy(m.data.data(), batch, rows * dim * 4);
        Changeset cs;
        cs.in_ids.assign(in_ids, in_ids + n_in);
        cs.in_positions.assign(in_pos, in_pos + n_in);
        cs.out_ids.assign(out_ids, out_ids + n_out);
        c.apply_changeset(m, std::span<const NodeId>(ids, n_ids), cs);
    });
}

int gxr_cache_resident(void* ch, uint64_t* out, uint64_t cap, uint64_t* n) {
    return guard([&] {
        auto r = static_cast<Cache*>(ch)->c->resident_set();
        *n = r.size();
        for (uint64_t i = 0; i < r.size() && i < cap; ++i) out[i] = r[i];
    });
}

int gxr_cache_row(void* ch, uint64_t v, float* out) {
    return guard([&] {
        auto r = static_cast<Cache*>(ch)->c->cached_row(v);
        std::memcpy(out, r.data(), r.size() * 4);
    });
}

// --- timed reference stages for bench.py (cpu_baseline / --impl reference) --

/// One superbatch through the reference's own stages, exactly as
/// TrainingRunner::run_superbatch (pipeline.hpp:338) sequences them but
/// without the compute stub: superbatch_sample (files) -> precompute_changesets
/// (files) -> FeatureCache ctor -> per iteration read ids/update files, gather,
/// apply_changeset. times[0..3] = sample, precompute, switch, main loop seconds.
int gxr_run_superbatch(const char* graph_path, const char* feature_path, const char* rt_dir,
                       const uint64_t* seeds_flat, const uint64_t* batch_off, uint64_t n_batches,
                       const uint32_t* fanouts, uint32_t n_layers, uint64_t global_seed,
                       uint64_t first_global_batch, uint64_t K, unsigned workers,
                       double* times, uint64_t* sampled_edges, uint64_t* gathered_rows,
                       uint64_t* total_misses) {
    return guard([&] {
        GraphFile g = GraphFile::open(graph_path);
        FeatureFile f = FeatureFile::open(feature_path);
        std::vector<std::vector<NodeId>> batches(n_batches);
        for (uint64_t b = 0; b < n_batches; ++b)
            batches[b].assign(seeds_flat + batch_off[b], seeds_flat + batch_off[b + 1]);
        Fanouts fo(fanouts, fanouts + n_layers);
        const uint64_t sb = 0;
        double t0 = now_s();
        superbatch_sample(g, nullptr, batches, fo, global_seed, first_global_batch, sb, rt_dir,
                          workers);
        double t1 = now_s();
        FileTrace tr;
        for (uint64_t i = 0; i < n_batches; ++i) tr.files.push_back(ids_file_path(rt_dir, sb, i));
        auto pr = precompute_changesets(tr, g.num_nodes(), K, rt_dir, sb);
        double t2 = now_s();
        IoStats io;
        auto init = read_init_file(init_file_path(rt_dir, sb));
        FeatureCache cache(f, init, K, io);
        double t3 = now_s();
        RowMatrix batch;
        uint64_t rows = 0, miss = 0, edges = 0;
        for (uint64_t i = 0; i < n_batches; ++i) {
            auto ids = read_ids_file(ids_file_path(rt_dir, sb, i));
            auto adj = read_adj_file(adj_file_path(rt_dir, sb, i));
            auto c = cache.gather(f, ids, batch, io);
            Changeset cs = read_update_file(update_file_path(rt_dir, sb, i));
            cache.apply_changeset(batch, ids, cs);
            rows += ids.size();
            miss += c.misses;
            for (auto& l : adj) edges += l.size();
        }
        double t4 = now_s();
        times[0] = t1 - t0;
        times[1] = t2 - t1;
        times[2] = t3 - t2;
        times[3] = t4 - t3;
        *sampled_edges = edges;
        *gathered_rows = rows;
        *total_misses = miss;
        (void)pr;
    });
}

/// run_training (pipeline.hpp:451): the whole TrainingRunner loop (sample,
/// precompute, executor with compute_stub) on the given files; returns every
/// iteration's checksum in order (StageMetrics::checksums, pipeline.hpp:426).
int gxr_run_training(const char* graph_path, const char* feature_path, const char* ncache_path,
                     const char* rt_dir, const uint32_t* fanouts, uint32_t n_layers, uint64_t batch_size,
                     uint64_t superbatch_size, uint64_t epochs, uint64_t cache_entries, int use_ncache,
                     int overlap, unsigned workers, uint64_t seed, double train_fraction, uint64_t* checksums,
                     uint64_t cap, uint64_t* n) {
    return guard([&] {
        RunConfig cfg;
        cfg.graph_path = graph_path;
        cfg.feature_path = feature_path;
        if (ncache_path) cfg.neighbor_cache_path = ncache_path;
        cfg.runtime_dir = rt_dir;
        cfg.fanouts.assign(fanouts, fanouts + n_layers);
        cfg.batch_size = batch_size;
        cfg.superbatch_size = superbatch_size;
        cfg.epochs = epochs;
        cfg.feature_cache_entries = cache_entries;
        cfg.use_neighbor_cache = use_ncache != 0;
        cfg.overlap = overlap != 0;
        cfg.sampler_workers = workers;
        cfg.seed = seed;
        cfg.train_fraction = train_fraction;
        RunReport r = run_training(cfg);
        uint64_t k = 0;
        for (auto& sb : r.superbatches)
            for (auto c : sb.checksums) {
                if (k < cap) checksums[k] = c;
                ++k;
            }
        *n = k;
    });
}

/// compute_stub (pipeline.hpp:35-57) over a batch and its adjacency
uint64_t gxr_compute_stub(const float* rows, uint64_t n_rows, uint32_t dim, const uint32_t* pairs,
                          const uint64_t* layer_counts, uint32_t n_layers) {
    RowMatrix batch;
    batch.resize(n_rows, dim);
    std::copy(rows, rows + n_rows * dim, batch.data.begin());
    std::vector<std::vector<LocalEdge>> adj(n_layers);
    uint64_t k = 0;
    for (uint32_t l = 0; l < n_layers; ++l)
        for (uint64_t e = 0; e < layer_counts[l]; ++e, ++k) adj[l].push_back({pairs[2 * k], pairs[2 * k + 1]});
    return compute_stub(batch, adj);
}

} // extern "C"
