// batch_pipeline.cpp — the batched C++ API (include/cdx/batch.hpp) end to end, as a C++
// serving host would drive it: synthetic traces generated on the device (cdx_gen_*), then
//   SC     sc_certaindex -> allocate_scan -> sc_aggregate   (also replayed as a batch::Graph)
//   CoT    cot_exit + cot_eps_stop
//   MCTS/Rebase  reward_certaindex -> reward_aggregate at each program's first met step
//   JSONL  jsonl_parse of a small trace
// Every output is written as a raw little-endian file into argv[1];
// tests/test_gpu_batch_cpp.py recomputes each one with the oracle and compares bit for bit.

#include <cstdint>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "cdx/batch.hpp"

using namespace cdx;

namespace {

std::string g_dir;

template <class T>
void dump(const std::string& name, const std::vector<T>& v) {
    std::ofstream f(g_dir + "/" + name + ".bin", std::ios::binary);
    f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(T)));
}

cdx_gen_params gen(uint64_t seed, uint32_t conv_hi, double hes) {
    cdx_gen_params g{};
    g.seed = seed;
    g.groups = 5;
    g.conv_lo = 1;
    g.conv_hi = conv_hi;
    g.noise_level = 0.5;
    g.residual_noise = 0.0;
    g.solvable_fraction = 0.9;
    g.hesitation_prob = hes;
    g.reward_start_k = 5033165;
    g.reward_final_k = 15099494;
    g.reward_unsolvable_k = 4194304;
    g.reward_jitter_k = 1677722;
    return g;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: batch_pipeline <out-dir>\n");
        return 2;
    }
    g_dir = argv[1];
    try {
        batch::Context cx(0);
        // ---- SC: 4096 requests x 64 probes x 32 samples
        {
            const uint64_t R = 4096;
            const uint32_t P = 64, S = 32;
            batch::DeviceArray<uint32_t> ids(cx, R * P * S);
            const auto g = gen(31, 64, 0.0);
            cx.check(cdx_gen_sc(cx.raw(), &g, 0, R, P, S, ids.data()));
            batch::DeviceArray<float> hc(cx, R * P);
            batch::DeviceArray<uint32_t> meets(cx, R * 2);
            const metrics::SignalThreshold th{metrics::SignalKind::CertaindexEntropy, 0.7};
            scheduler::AllocationPolicy pol;
            pol.kind = scheduler::AllocationKind::StaticThreshold;
            pol.detect_at_knob = 5;
            pol.resource_cap = 64;
            batch::DeviceArray<int32_t> ek(cx, R), gr(cx, R);
            batch::DeviceArray<uint8_t> why(cx, R);
            batch::DeviceArray<int64_t> off(cx, R), sc(cx, 3);
            batch::DeviceArray<uint32_t> kept(cx, R), ans(cx, R);
            batch::AllocationOutputs o{ek.data(), why.data(), gr.data(), off.data(), kept.data(),
                                       reinterpret_cast<uint64_t*>(sc.data()), sc.data() + 1, sc.data() + 2};
            auto step = [&] {
                batch::sc_certaindex(cx, ids.data(), {R, P, S}, {&th, 1}, hc.data(), meets.data());
                batch::allocate_scan(cx, meets.data(), R, P, pol, 64 * S, 0, 0, o);
                batch::sc_aggregate(cx, ids.data(), {R, P, S}, ek.data(), ans.data());
            };
            step();
            cx.sync();
            dump("sc_hcert", hc.download());
            dump("sc_meets", meets.download());
            dump("sc_exit", ek.download());
            dump("sc_offsets", off.download());
            dump("sc_answer", ans.download());
            dump("sc_scalars", sc.download());
            // the same step captured once and replayed twice
            ek.zero();
            ans.zero();
            batch::Graph graph(cx, step);
            graph.launch();
            graph.launch();
            cx.sync();
            dump("sc_exit_graph", ek.download());
            dump("sc_answer_graph", ans.download());
            // majority-fraction certaindex ANDed with the entropy threshold
            batch::DeviceArray<float> mj(cx, R * P);
            const batch::MajorityThreshold mt{0.6, metrics::ThresholdDir::GreaterEq};
            batch::sc_certaindex(cx, ids.data(), {R, P, S}, {&th, 1}, {&mt, 1}, nullptr, mj.data(), meets.data());
            cx.sync();
            dump("sc_majority", mj.download());
            dump("sc_meets_majority", meets.download());
        }
        // ---- CoT: 8192 requests x 64 probes, w = 3, tau = 0.9, budget at the last probe
        {
            const uint64_t R = 8192;
            const uint32_t P = 64;
            batch::DeviceArray<uint32_t> ids(cx, R * P);
            batch::DeviceArray<uint64_t> hes(cx, R);
            const auto g = gen(32, 64, 0.05);
            cx.check(cdx_gen_cot(cx.raw(), &g, 0, R, P, ids.data(), hes.data()));
            probe::ProbeConfig cfg;
            cfg.max_tokens = 4096;
            batch::DeviceArray<int32_t> ex(cx, R), eps(cx, R);
            batch::DeviceArray<uint8_t> why(cx, R), low(cx, R);
            batch::DeviceArray<uint32_t> fid(cx, R);
            batch::cot_exit(cx, ids.data(), hes.data(), nullptr, R, P, cfg,
                            {ex.data(), why.data(), fid.data(), low.data(), nullptr});
            batch::cot_eps_stop(cx, ids.data(), hes.data(), R, P, 3, 0.5, eps.data(), nullptr);
            dump("cot_exit", ex.download());
            dump("cot_reason", why.download());
            dump("cot_final", fid.download());
            dump("cot_eps", eps.download());
        }
        // ---- MCTS (even) / Rebase (odd): 2048 programs x 16 steps x 64 nodes
        {
            const uint64_t G = 2048;
            const uint32_t T = 16, W = 64;
            batch::DeviceArray<float> rw(cx, G * T * W);
            batch::DeviceArray<uint32_t> ids(cx, G * T * W);
            const auto g = gen(33, 16, 0.0);
            cx.check(cdx_gen_reward(cx.raw(), &g, 0, G, T, W, rw.data(), ids.data()));
            std::vector<uint8_t> agg(G);
            for (uint64_t i = 0; i < G; ++i) agg[i] = static_cast<uint8_t>(i % 2);
            batch::DeviceArray<uint8_t> d_agg(cx, std::span<const uint8_t>(agg));
            const metrics::SignalThreshold tm[2] = {{metrics::SignalKind::CertaindexEntropy, 0.99},
                                                    {metrics::SignalKind::CertaindexReward, 0.4}};
            const metrics::SignalThreshold tx[2] = {{metrics::SignalKind::CertaindexEntropy, 0.85},
                                                    {metrics::SignalKind::CertaindexReward, 0.99}};
            batch::DeviceArray<float> Rv(cx, G * T), Hv(cx, G * T);
            batch::DeviceArray<uint32_t> m(cx, G);
            batch::reward_certaindex(cx, rw.data(), ids.data(), d_agg.data(), G, T, W, tm, tx, Rv.data(), Hv.data(),
                                     m.data());
            const auto mh = m.download();
            std::vector<int32_t> step(G);
            for (uint64_t i = 0; i < G; ++i) step[i] = mh[i] ? __builtin_ctz(mh[i]) : static_cast<int32_t>(T - 1);
            batch::DeviceArray<int32_t> d_step(cx, std::span<const int32_t>(step));
            batch::DeviceArray<uint32_t> ans(cx, G);
            const uint64_t inexact =
                batch::reward_aggregate(cx, rw.data(), ids.data(), d_agg.data(), G, T, W, d_step.data(), ans.data());
            dump("rw_R", Rv.download());
            dump("rw_H", Hv.download());
            dump("rw_meets", mh);
            dump("rw_answer", ans.download());
            dump("rw_inexact", std::vector<uint64_t>{inexact});
        }
        // ---- JSONL
        {
            const std::string text =
                "{\"program_id\":\"a\",\"step_index\":1,\"token_offset\":64,\"answer\":\" 12 \"}\n"
                "\n"
                "{\"program_id\":\"b\",\"step_index\":1,\"token_offset\":64,\"answer\":\"wait, 7\",\"hesitant\":true}\n"
                "{\"program_id\":\"a\",\"step_index\":2,\"token_offset\":128,\"answer\":\"12\"}\n";
            batch::DeviceArray<char> d(cx, std::span<const char>(text.data(), text.size()));
            const uint64_t cap = 8;
            batch::DeviceArray<uint32_t> pg(cx, cap);
            batch::DeviceArray<int32_t> st(cx, cap);
            batch::DeviceArray<int64_t> tk(cx, cap);
            batch::DeviceArray<uint8_t> hs(cx, cap);
            batch::DeviceArray<uint64_t> ao(cx, cap + 1);
            batch::DeviceArray<char> aa(cx, text.size());
            batch::JsonlRecords o;
            o.program = pg.data();
            o.step_index = st.data();
            o.token_offset = tk.data();
            o.hesitant = hs.data();
            o.answer_off = ao.data();
            o.answer_arena = aa.data();
            const auto [nr, np] = batch::jsonl_parse(cx, d.data(), text.size(), cap, o);
            dump("jl_counts", std::vector<uint64_t>{nr, np});
            dump("jl_program", pg.download());
            dump("jl_step", st.download());
            dump("jl_tok", tk.download());
            dump("jl_hes", hs.download());
            dump("jl_answer_off", ao.download());
            dump("jl_answer_arena", aa.download());
        }
        std::printf("batch_pipeline: ok (%llu kernel launches)\n", static_cast<unsigned long long>(cx.launches()));
        return 0;
    } catch (const std::exception& e) {
        std::printf("batch_pipeline: EXC %s\n", e.what());
        return 1;
    }
}
