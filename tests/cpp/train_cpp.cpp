// C++ consumer of the reference-shaped API (include/ember/{model,config,pipeline}.h) — what the
// reference's own C++ (proj/, namespace ember) would write against the B200 library. Used by
// tests/test_cpp_api.py:
//   train_cpp cpu            RunConfig validation + score() known answers (no GPU needed)
//   train_cpp gpu <outdir>   one batch through the per-op API (sample_negatives -> loss_and_grad ->
//                            adagrad_step), then a train_epoch_sync epoch and a train_epoch_partitioned
//                            epoch through the partition buffer (p=4, c=2); arrays written to <outdir>
//                            for comparison with the CPU oracle.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "ember/config.h"
#include "ember/model.h"
#include "ember/pipeline.h"

using namespace ember;

static int fails = 0;
#define EXPECT(c)                                                         \
    do {                                                                  \
        if (!(c)) {                                                       \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++fails;                                                      \
        }                                                                 \
    } while (0)

template <typename F>
static bool throws_config(F&& f) {
    try {
        f();
    } catch (const ConfigError&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

template <typename T>
static void dump(const std::string& dir, const std::string& name, const std::vector<T>& v) {
    std::ofstream f(dir + "/" + name + ".bin", std::ios::binary);
    f.write(reinterpret_cast<const char*>(v.data()), (std::streamsize)(v.size() * sizeof(T)));
}

static int cpu_checks() {
    // score known answers
    EXPECT(score(ModelKind::Dot, {1, 2}, {}, {3, 4}) == 11.f);
    const std::vector<float> s{0.5f, -1.f, 2.f, 0.25f}, d{1.5f, 2.f, -0.5f, 4.f}, ones(4, 1.f);
    EXPECT(score(ModelKind::DistMult, s, ones, d) == score(ModelKind::Dot, s, {}, d));
    const std::vector<float> sc{0.5f, -1.f, 0.f, 0.f}, rc{2.f, 3.f, 0.f, 0.f}, dc{1.5f, 2.f, 0.f, 0.f};
    EXPECT(score(ModelKind::ComplEx, sc, rc, dc) ==
           score(ModelKind::DistMult, {0.5f, -1.f}, {2.f, 3.f}, {1.5f, 2.f}));
    EXPECT(throws_config([] { score(ModelKind::Dot, {1, 2}, {}, {3}); }));
    EXPECT(model_kind_from_string("complex") == ModelKind::ComplEx && to_string(ModelKind::Dot) == "dot");
    EXPECT(throws_config([] { model_kind_from_string("transe"); }));
    // RunConfig validation: violations are ConfigErrors before any device work
    RunConfig ok;
    ok.validate();
    auto bad = [&](auto mutate) {
        RunConfig c = ok;
        mutate(c);
        return throws_config([&] { c.validate(); });
    };
    EXPECT(bad([](RunConfig& c) { c.dim = 0; }));
    EXPECT(bad([](RunConfig& c) { c.dim = 102; }));
    EXPECT(bad([](RunConfig& c) { c.eps = 0.f; }));
    EXPECT(bad([](RunConfig& c) { c.negatives.alpha = 1.5f; }));
    EXPECT(bad([](RunConfig& c) { c.staleness_bound = 0; }));
    EXPECT(bad([](RunConfig& c) { c.num_partitions = 4; }));  // in-memory needs p = 1
    EXPECT(bad([](RunConfig& c) {
        c.backend = StorageBackend::Partitioned;
        c.num_partitions = 4;
        c.buffer_capacity = 1;
    }));
    EXPECT(bad([](RunConfig& c) {
        c.backend = StorageBackend::Partitioned;
        c.num_partitions = 4;
        c.buffer_capacity = 5;
    }));
    RunConfig part = ok;
    part.backend = StorageBackend::Partitioned;
    part.num_partitions = 16;
    part.buffer_capacity = 4;
    part.validate();
    std::printf("cpu ok (%d failures)\n", fails);
    return fails ? 1 : 0;
}

static int gpu_run(const std::string& out) {
    const uint64_t V = 3000, E = 20000;
    const uint32_t R = 20;
    std::vector<uint32_t> raw(3 * E);
    std::vector<uint8_t> split(E);
    gpu::check(ember_graph_generate(-1, V, R, E, 5, 0.9f, 0.05f, raw.data(), split.data()));
    std::vector<uint32_t> train;
    for (uint64_t e = 0; e < E; ++e)
        if (split[e] == 0) train.insert(train.end(), &raw[3 * e], &raw[3 * e + 3]);
    const uint64_t n = train.size() / 3;
    std::printf("train edges %llu\n", (unsigned long long)n);

    RunConfig cfg;
    cfg.model = ModelKind::ComplEx;
    cfg.dim = 32;
    cfg.batch_size = 256;
    cfg.negatives.n_t = 64;
    cfg.negatives.seed = 3;
    cfg.backend = StorageBackend::Partitioned;
    cfg.num_partitions = 2;
    cfg.buffer_capacity = 2;  // c = p: every partition resident in HBM
    cfg.init_seed = 11;

    std::vector<uint32_t> bucketed(3 * n);
    std::vector<uint64_t> off(5);
    gpu::check(ember_graph_bucket(-1, V, 2, train.data(), n, bucketed.data(), off.data()));
    dump(out, "edges_p2", bucketed);
    dump(out, "offsets_p2", off);
    {
        Trainer tr(cfg, V, R);
        gpu::Context& ctx = tr.context();
        tr.init_embeddings();
        dump(out, "theta0_p0", tr.download(0));
        dump(out, "theta0_p1", tr.download(1));
        dump(out, "rel0", tr.download(EMBER_RELATIONS));
        DeviceArray<uint32_t> dev(ctx, bucketed);
        // one batch of bucket (0, 1) through the per-op API
        const uint32_t* b01 = dev.data() + 3 * off[1];
        const uint64_t n01 = off[2] - off[1];
        auto negs = sample_negatives(ctx, cfg.negatives, b01, n01, 0, 1, 0, 0, 0);
        LossAndGrad lg = loss_and_grad(ctx, cfg.dim, b01, cfg.batch_size, 0, 1, negs.data(), negs.size());
        EXPECT(std::isfinite(lg.loss));
        dump(out, "negs", negs.download());
        dump(out, "fpos", lg.fpos.download());
        dump(out, "lse", lg.lse.download());
        dump(out, "node_ids", lg.delta.node_ids.download(lg.delta.n_nodes));
        dump(out, "node_rows", lg.delta.node_rows.download((size_t)lg.delta.n_nodes * cfg.dim));
        dump(out, "rel_ids", lg.delta.rel_ids.download(lg.delta.n_rels));
        dump(out, "rel_rows", lg.delta.rel_rows.download((size_t)lg.delta.n_rels * cfg.dim));
        dump(out, "loss", std::vector<double>{lg.loss});
        adagrad_step(ctx, lg.delta, 0, 1);
        dump(out, "theta1_p0", tr.download(0));
        dump(out, "theta1_p1", tr.download(1));
        dump(out, "acc1_p0", tr.download(0, true));
        dump(out, "acc1_p1", tr.download(1, true));
        dump(out, "rel1", tr.download(EMBER_RELATIONS));
        // a whole epoch (Algorithm 1 over the plan's buckets)
        EpochStats st = train_epoch_sync(tr, dev.data(), off, 0);
        EXPECT(st.edges == n && st.batches > 0 && std::isfinite(st.mean_loss));
        dump(out, "epoch_loss_p2", std::vector<double>{st.mean_loss});
        dump(out, "theta2_p0", tr.download(0));
        dump(out, "theta2_p1", tr.download(1));
        dump(out, "rel2", tr.download(EMBER_RELATIONS));
    }
    {   // train_epoch_partitioned through the device partition buffer: p = 4, c = 2
        RunConfig pc = cfg;
        pc.num_partitions = 4;
        std::vector<uint32_t> b4(3 * n);
        std::vector<uint64_t> off4(17);
        gpu::check(ember_graph_bucket(-1, V, 4, train.data(), n, b4.data(), off4.data()));
        dump(out, "edges_p4", b4);
        dump(out, "offsets_p4", off4);
        std::vector<uint32_t> seq;
        for (int c : {2, 4}) {
            pc.buffer_capacity = c;
            Trainer tr(pc, V, R);
            EXPECT(tr.buffered() == (c < 4));
            if (c == 4) tr.use_plan(make_plan(OrderingKind::Elimination, 4, 2, 0));  // the buffered run's order
            tr.init_embeddings();
            DeviceArray<uint32_t> dev(tr.context(), b4);
            EpochStats a = train_epoch_partitioned(tr, dev.data(), off4, 0);
            EpochStats b = train_epoch_partitioned(tr, dev.data(), off4, 1);
            if (c == 2) {
                EXPECT(a.buffer_reads == 2 + tr.plan().swap_count && b.buffer_reads == a.buffer_reads);
                for (const BucketId& x : tr.plan().bucket_sequence) {
                    seq.push_back(x.i);
                    seq.push_back(x.j);
                }
                dump(out, "plan_p4c2", seq);
            }
            std::vector<float> all;
            for (uint32_t k = 0; k < 4; ++k) {
                auto t = tr.download(k);
                all.insert(all.end(), t.begin(), t.end());
            }
            dump(out, "theta_p4_c" + std::to_string(c), all);
            dump(out, "rel_p4_c" + std::to_string(c), tr.download(EMBER_RELATIONS));
            dump(out, "loss_p4_c" + std::to_string(c), std::vector<double>{a.mean_loss, b.mean_loss});
        }
    }
    std::printf("gpu ok (%d failures)\n", fails);
    return fails ? 1 : 0;
}

int main(int argc, char** argv) {
    try {
        if (argc >= 2 && std::string(argv[1]) == "cpu") return cpu_checks();
        if (argc >= 3 && std::string(argv[1]) == "gpu") return gpu_run(argv[2]);
        std::fprintf(stderr, "usage: train_cpp cpu | gpu <outdir>\n");
        return 2;
    } catch (const EmberError& e) {
        std::fprintf(stderr, "EmberError: %s\n", e.what());
        return 3;
    }
}
