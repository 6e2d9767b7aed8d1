// ref_bench.cpp — times the UNMODIFIED reference CPU forward
// (Model<float>::forward_sample, proj/include/mtfm/model.hpp:251-312) over a
// generated batch, users striped over std::thread workers exactly like the
// reference's own parallel scoring (Trainer::records_of,
// proj/include/mtfm/train.hpp:157-170).
//
// TEST / BASELINE INFRASTRUCTURE ONLY: used by bench.py's cpu_baseline leg and
// by `bench.py --impl reference`. Prints one JSON line per rep.
//
// --batch FILE [--params FILE]: score the users of an MTFMPB1 packed batch (the
// GPU arm's own input bytes, paper_2602_11235_b200/packed_io.py) with the
// model config stored in it and, optionally, the GPU arm's parameters;
// --users N limits the sample to the file's first N users. Without --batch the
// reference generator (datagen.cpp) makes the users.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <iostream>
#include <string>
#include <thread>
#include <vector>

#include "mtfm/datagen.hpp"
#include "mtfm/model.hpp"
#include "packed_io.hpp"

using namespace mtfm;

int main(int argc, char** argv) {
    GeneratorConfig gc;
    gc.n_scenarios = 4;
    gc.n_users = 32;
    gc.n_hist_seqs = 2;
    gc.n_rt_seqs = 1;
    gc.seq_len_min = 224;
    gc.seq_len_max = 224;
    gc.exposures_min = 8;
    gc.exposures_max = 8;
    gc.seed = 3;
    ModelConfig mc;
    mc.hta.d_model = 256;
    mc.hta.blocks = 1;
    mc.hta.target_layers = 3;
    mc.hta.full_layers = 1;
    mc.hta.heads = 8;
    mc.hta.kv_heads = 2;
    mc.d_emb = 16;
    mc.experts = 4;
    mc.d_expert = 256;
    int threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    int reps = 1, rlen = -1;
    std::string batch_file, params_file;
    bool users_set = false;
    try {
        for (int i = 1; i < argc; ++i) {
            std::string a = argv[i];
            auto nxt = [&]() -> std::string {
                if (i + 1 >= argc) throw config_error("missing value for " + a);
                return argv[++i];
            };
            if (a == "--users") {
                gc.n_users = std::stoi(nxt());
                users_set = true;
            }
            else if (a == "--scen") gc.n_scenarios = std::stoi(nxt());
            else if (a == "--nh") gc.n_hist_seqs = std::stoi(nxt());
            else if (a == "--nr") gc.n_rt_seqs = std::stoi(nxt());
            else if (a == "--lenmin") gc.seq_len_min = std::stoi(nxt());
            else if (a == "--lenmax") gc.seq_len_max = std::stoi(nxt());
            else if (a == "--expmin") gc.exposures_min = std::stoi(nxt());
            else if (a == "--expmax") gc.exposures_max = std::stoi(nxt());
            else if (a == "--gseed") gc.seed = std::stoull(nxt());
            else if (a == "--rlen") rlen = std::stoi(nxt());
            else if (a == "--d") mc.hta.d_model = std::stoi(nxt());
            else if (a == "--blocks") mc.hta.blocks = std::stoi(nxt());
            else if (a == "--K") mc.hta.target_layers = std::stoi(nxt());
            else if (a == "--P") mc.hta.full_layers = std::stoi(nxt());
            else if (a == "--H") mc.hta.heads = std::stoi(nxt());
            else if (a == "--G") mc.hta.kv_heads = std::stoi(nxt());
            else if (a == "--dexp") mc.d_expert = std::stoi(nxt());
            else if (a == "--threads") threads = std::stoi(nxt());
            else if (a == "--reps") reps = std::stoi(nxt());
            else if (a == "--batch") batch_file = nxt();
            else if (a == "--params") params_file = nxt();
            else throw config_error("unknown flag " + a);
        }
        Dataset d;
        if (!batch_file.empty()) {
            mtfa::PackedFile pf = mtfa::load_packed(batch_file);
            if (pf.has_model) mc = pf.cfg;
            d = std::move(pf.data);
            if (users_set && gc.n_users < static_cast<int>(d.samples.size())) d.samples.resize(static_cast<size_t>(gc.n_users));
        } else {
            d = generate_dataset(gc);
        }
        if (rlen >= 0 && batch_file.empty())
            for (auto& s : d.samples)
                for (auto& rec : s.realtime_sequences)
                    if (static_cast<int>(rec.events.size()) > rlen) rec.events.resize(static_cast<size_t>(rlen));
        Model<float> model = Model<float>::build(SchemaSet::from(d), mc, 7);
        if (!params_file.empty()) mtfa::load_params_into(params_file, model.params);
        size_t targets = 0, tokens = 0;
        for (const auto& s : d.samples) {
            targets += s.exposures.size();
            tokens += s.exposures.size();
            for (const auto& r : s.historical_sequences) tokens += r.events.size();
            for (const auto& r : s.realtime_sequences) tokens += r.events.size();
        }
        for (int rep = 0; rep < reps; ++rep) {
            std::atomic<size_t> n_records{0};
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> pool;
            for (int w = 0; w < threads; ++w) {
                pool.emplace_back([&, w]() {
                    size_t local = 0;
                    for (size_t u = static_cast<size_t>(w); u < d.samples.size(); u += static_cast<size_t>(threads))
                        local += model.forward_sample(d.samples[u]).size();
                    n_records += local;
                });
            }
            for (auto& t : pool) t.join();
            auto t1 = std::chrono::steady_clock::now();
            double secs = std::chrono::duration<double>(t1 - t0).count();
            std::printf(
                "{\"rep\": %d, \"seconds\": %.6f, \"users\": %zu, \"targets\": %zu, \"tokens\": %zu, "
                "\"records\": %zu, \"threads\": %d, \"targets_per_sec\": %.3f, \"tokens_per_sec\": %.3f}\n",
                rep, secs, d.samples.size(), targets, tokens, n_records.load(), threads,
                static_cast<double>(targets) / secs, static_cast<double>(tokens) / secs);
            std::fflush(stdout);
        }
    } catch (const std::exception& e) {
        std::cerr << "ref_bench: " << e.what() << "\n";
        return 1;
    }
    return 0;
}
