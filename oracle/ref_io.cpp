// ref_io.cpp — golden vectors for dataset ingestion, produced by the UNMODIFIED
// reference dataset I/O (proj/src/dataset_io.cpp, nlohmann/json 3.11.3).
//
// TEST INFRASTRUCTURE ONLY.
//   ref_io gen OUT.jsonl USERS SEED   generate_dataset + save_dataset
//   ref_io load IN.jsonl OUT.mtfa     load_dataset -> packed arrays + labels, or the
//                                     exception class and what() it throws
#include <iostream>
#include <string>
#include <vector>

#include "mtfa.hpp"
#include "mtfm/dataset_io.hpp"
#include "mtfm/datagen.hpp"

using namespace mtfm;

int main(int argc, char** argv) {
    if (argc < 4) {
        std::cerr << "usage: ref_io gen OUT USERS SEED | ref_io load IN OUT\n";
        return 2;
    }
    const std::string mode = argv[1];
    if (mode == "gen") {
        GeneratorConfig gc;
        gc.n_scenarios = 4;
        gc.n_users = argc > 3 ? std::stoi(argv[3]) : 40;
        gc.seed = argc > 4 ? std::stoull(argv[4]) : 1;
        gc.seq_len_min = 0;
        gc.seq_len_max = 30;
        gc.exposures_min = 0;
        gc.exposures_max = 5;
        save_dataset(generate_dataset(gc), argv[2]);
        return 0;
    }
    mtfa::Writer w(argv[3]);
    std::string kind, what;
    try {
        Dataset d = load_dataset(argv[2]);
        int max_tasks = 0;
        for (const auto& s : d.scenarios) max_tasks = std::max(max_tasks, static_cast<int>(s.tasks.size()));
        std::vector<int64_t> user_id, ev_ts, exp_ts;
        std::vector<int32_t> seq_off{0}, seq_schema, ev_off{0}, ev_feat_off{0}, ev_feats, exp_off{0}, exp_scen,
            exp_feat_off{0}, exp_blk, exp_feats, labels;
        std::vector<uint8_t> seq_kind;
        for (const auto& s : d.samples) {
            user_id.push_back(s.user_id);
            auto eat = [&](const std::vector<SequenceRecord>& v, uint8_t k) {
                for (const auto& rec : v) {
                    seq_kind.push_back(k);
                    seq_schema.push_back(rec.seq_schema_id);
                    for (const auto& ev : rec.events) {
                        ev_ts.push_back(ev.timestamp);
                        for (int f : ev.item_features) ev_feats.push_back(f);
                        ev_feat_off.push_back(static_cast<int32_t>(ev_feats.size()));
                    }
                    ev_off.push_back(static_cast<int32_t>(ev_ts.size()));
                }
            };
            eat(s.historical_sequences, 0);
            eat(s.realtime_sequences, 1);
            seq_off.push_back(static_cast<int32_t>(seq_kind.size()));
            for (const auto& e : s.exposures) {
                exp_scen.push_back(e.scenario_id);
                exp_ts.push_back(e.timestamp);
                exp_blk.push_back(static_cast<int32_t>(e.user_features.size()));
                exp_blk.push_back(static_cast<int32_t>(e.cross_features.size()));
                exp_blk.push_back(static_cast<int32_t>(e.item_features.size()));
                for (int f : e.user_features) exp_feats.push_back(f);
                for (int f : e.cross_features) exp_feats.push_back(f);
                for (int f : e.item_features) exp_feats.push_back(f);
                exp_feat_off.push_back(static_cast<int32_t>(exp_feats.size()));
                const auto& tasks = d.scenario(e.scenario_id).tasks;
                for (int t = 0; t < max_tasks; ++t) {
                    int v = -1;
                    if (t < static_cast<int>(tasks.size())) {
                        auto it = e.labels.find(tasks[static_cast<size_t>(t)]);
                        if (it != e.labels.end()) v = it->second;
                    }
                    labels.push_back(v);
                }
            }
            exp_off.push_back(static_cast<int32_t>(exp_scen.size()));
        }
        w.put("user_id", user_id);
        w.put("seq_off", seq_off);
        w.put("seq_kind", seq_kind);
        w.put("seq_schema", seq_schema);
        w.put("ev_off", ev_off);
        w.put("ev_ts", ev_ts);
        w.put("ev_feat_off", ev_feat_off);
        w.put("ev_feats", ev_feats);
        w.put("exp_off", exp_off);
        w.put("exp_scenario", exp_scen);
        w.put("exp_ts", exp_ts);
        w.put("exp_feat_off", exp_feat_off);
        w.put("exp_blk", exp_blk);
        w.put("exp_feats", exp_feats);
        w.put("labels", labels);
        w.put("max_tasks", std::vector<int32_t>{max_tasks});
        kind = "ok";
    } catch (const parse_error& e) {
        kind = "parse_error", what = e.what();
    } catch (const config_error& e) {
        kind = "config_error", what = e.what();
    } catch (const integrity_error& e) {
        kind = "integrity_error", what = e.what();
    } catch (const lookup_error& e) {
        kind = "lookup_error", what = e.what();
    } catch (const std::exception& e) {
        kind = "other", what = e.what();
    }
    w.put_str("kind", kind);
    w.put_str("what", what);
    return 0;
}
