// Reference unit tests restated against the C++ adapter (include/gx_b200.hpp):
// the same calls a reference user makes, now landing on the B200 kernels.
// Built by tests/test_cpp_adapter.py (CPU: compile+link; GPU: run).
#include <cassert>
#include <cstdio>
#include <map>
#include <set>

#include "gx_b200.hpp"

using namespace gx_b200;

struct MemoryTrace {  // changeset.hpp:44-48
    const std::vector<std::vector<NodeId>>* trace;
    std::size_t iterations() const { return trace->size(); }
    std::vector<NodeId> ids(std::size_t i) const { return (*trace)[i]; }
};

#define REQUIRE(c)                                                     \
    do {                                                               \
        if (!(c)) {                                                    \
            std::fprintf(stderr, "FAILED %s:%d %s\n", __FILE__, __LINE__, #c); \
            return 1;                                                  \
        }                                                              \
    } while (0)

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: adapter_test <dir with graph.bin features.bin>\n");
        return 2;
    }
    const std::filesystem::path dir = argv[1];
    // test_changeset.cpp:150-171 (Fig. 11)
    std::vector<std::vector<NodeId>> t{{0, 2, 5, 7}, {1, 2, 4, 5, 7}, {6}};
    MemoryTrace mt{&t};
    AccessIndex ix = build_access_index(mt, 10);
    std::vector<NodeId> init{0, 1, 4, 6, 7};
    std::vector<Changeset> css;
    std::vector<std::vector<NodeId>> states;
    simulate_changesets(ix, mt, 5, init, [&](std::size_t, const Changeset& cs, std::span<const NodeId> st) {
        css.push_back(cs);
        states.emplace_back(st.begin(), st.end());
    });
    REQUIRE((css[0].in_ids == std::vector<NodeId>{2, 5}));
    REQUIRE((css[0].in_positions == std::vector<std::uint64_t>{1, 2}));
    REQUIRE((css[0].out_ids == std::vector<NodeId>{0, 6}));
    REQUIRE((states[0] == std::vector<NodeId>{1, 2, 4, 5, 7}));
    // test_changeset.cpp:143-148
    std::vector<std::vector<NodeId>> t2{{4, 1}, {2, 4, 9}};
    REQUIRE((compute_init_set(MemoryTrace{&t2}, 3, 10) == std::vector<NodeId>{4, 1, 2}));
    // errors keep their reference types (test_changeset.cpp:72-79)
    std::vector<std::vector<NodeId>> dup{{1, 1}};
    bool threw = false;
    try {
        build_access_index(MemoryTrace{&dup}, 3);
    } catch (const std::logic_error&) {
        threw = true;
    }
    REQUIRE(threw);
    // sampling invariants (test_sampler.cpp:92-134) on a reference-written graph.bin
    GraphFile g = GraphFile::open(dir / "graph.bin");
    IoStats s;
    std::vector<NodeId> seeds{1, 7, 42, 99};
    SampleOutput out = sample_batch(g, nullptr, seeds, {5, 5}, 11, s);
    REQUIRE(out.num_seeds == 4);
    std::set<NodeId> uniq(out.ids.begin(), out.ids.end());
    REQUIRE(uniq.size() == out.ids.size());
    REQUIRE(s.neighbor_lists_read > 0);
    // executor (test_feature_cache.cpp:55-71)
    FeatureFile f = FeatureFile::open(dir / "features.bin");
    IoStats io;
    std::vector<NodeId> cinit{0, 1, 4, 6, 7};
    FeatureCache c(f, cinit, 5, io);
    std::vector<NodeId> ids{0, 2, 5, 7};
    RowMatrix batch;
    auto counts = c.gather(f, ids, batch, io);
    REQUIRE(counts.hits == 2 && counts.misses == 2);
    Changeset cs;
    cs.in_ids = {2, 5};
    cs.in_positions = {1, 2};
    cs.out_ids = {0, 6};
    c.apply_changeset(batch, ids, cs);
    REQUIRE((c.resident_set() == std::vector<NodeId>{1, 2, 4, 5, 7}));
    REQUIRE(c.cached_row(5) == std::vector<float>(batch.row(2).begin(), batch.row(2).end()));
    std::printf("adapter_test: all checks passed\n");
    return 0;
}
