// ref_agg.cpp — golden vectors for user-level aggregation, produced by the
// UNMODIFIED reference aggregate_users (proj/src/datagen.cpp:171-216).
//
// TEST INFRASTRUCTURE ONLY. Writes an MTFA archive (oracle/mtfa.hpp) with, per
// case c<k>: the exposure stream in arrival order, the shared H/R store (the
// std::map flattened in iteration order), the scenario ids of the schema
// context, and either the reference's aggregated UserSamples in the packed
// jagged layout (+ its AggregationReport) or the integrity_error it throws.
// Cases: a generated dataset's exposures re-streamed in a seeded shuffle with
// extra store users that have no exposures; the worked cases of
// proj/tests/test_schema_data.cpp:122-147; the unknown-user / unknown-scenario
// failures of test_schema_data.cpp:150-173 (first offending element wins).
#include <algorithm>
#include <iostream>
#include <map>
#include <string>
#include <vector>

#include "mtfa.hpp"
#include "mtfm/datagen.hpp"
#include "mtfm/rng.hpp"
#include "mtfm/schema.hpp"

using namespace mtfm;

namespace {

struct Stream {
    std::vector<std::pair<int64_t, Exposure>> pairs;
};

void put_stream(mtfa::Writer& w, const std::string& p, const Stream& s) {
    std::vector<int64_t> uid, ts;
    std::vector<int32_t> sc, foff{0}, blk, feats;
    for (const auto& [u, e] : s.pairs) {
        uid.push_back(u);
        sc.push_back(e.scenario_id);
        ts.push_back(e.timestamp);
        blk.push_back(static_cast<int32_t>(e.user_features.size()));
        blk.push_back(static_cast<int32_t>(e.cross_features.size()));
        blk.push_back(static_cast<int32_t>(e.item_features.size()));
        for (int f : e.user_features) feats.push_back(f);
        for (int f : e.cross_features) feats.push_back(f);
        for (int f : e.item_features) feats.push_back(f);
        foff.push_back(static_cast<int32_t>(feats.size()));
    }
    w.put(p + "stream/user_id", uid);
    w.put(p + "stream/scenario", sc);
    w.put(p + "stream/ts", ts);
    w.put(p + "stream/feat_off", foff);
    w.put(p + "stream/blk", blk);
    w.put(p + "stream/feats", feats);
}

// packed jagged batch (include/mtfm_cuda.h layout) of samples, sequences only or all
void put_samples(mtfa::Writer& w, const std::string& p, const std::vector<UserSample>& ss) {
    std::vector<int64_t> user_id, ev_ts, exp_ts;
    std::vector<int32_t> seq_off{0}, seq_schema, ev_off{0}, ev_feat_off{0}, ev_feats, exp_off{0}, exp_scen,
        exp_feat_off{0}, exp_blk, exp_feats;
    std::vector<uint8_t> seq_kind;
    for (const auto& s : ss) {
        user_id.push_back(s.user_id);
        auto eat = [&](const std::vector<SequenceRecord>& seqs, uint8_t kind) {
            for (const auto& rec : seqs) {
                seq_kind.push_back(kind);
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
        }
        exp_off.push_back(static_cast<int32_t>(exp_scen.size()));
    }
    w.put(p + "user_id", user_id);
    w.put(p + "seq_off", seq_off);
    w.put(p + "seq_kind", seq_kind);
    w.put(p + "seq_schema", seq_schema);
    w.put(p + "ev_off", ev_off);
    w.put(p + "ev_ts", ev_ts);
    w.put(p + "ev_feat_off", ev_feat_off);
    w.put(p + "ev_feats", ev_feats);
    w.put(p + "exp_off", exp_off);
    w.put(p + "exp_scenario", exp_scen);
    w.put(p + "exp_ts", exp_ts);
    w.put(p + "exp_feat_off", exp_feat_off);
    w.put(p + "exp_blk", exp_blk);
    w.put(p + "exp_feats", exp_feats);
}

void run_case(mtfa::Writer& w, int k, const Dataset& ctx, const Stream& st, const std::map<int64_t, UserContext>& store) {
    const std::string p = "c" + std::to_string(k) + "/";
    put_stream(w, p, st);
    std::vector<UserSample> flat;
    for (const auto& [uid, c] : store) {
        UserSample s;
        s.user_id = uid;
        s.historical_sequences = c.historical;
        s.realtime_sequences = c.realtime;
        flat.push_back(std::move(s));
    }
    put_samples(w, p + "store/", flat);
    std::vector<int32_t> ids;
    for (const auto& s : ctx.scenarios) ids.push_back(s.scenario_id);
    std::sort(ids.begin(), ids.end());
    w.put(p + "scen_ids", ids);
    try {
        AggregationReport rep;
        auto out = aggregate_users(ctx, st.pairs, store, &rep);
        put_samples(w, p + "out/", out);
        w.put(p + "report", std::vector<int64_t>{static_cast<int64_t>(rep.n_exposure_records),
                                                 static_cast<int64_t>(rep.n_user_samples)});
        w.put(p + "ratio", std::vector<double>{rep.compression_ratio});
        w.put_str(p + "error", "");
    } catch (const integrity_error& e) {
        w.put_str(p + "error", e.what());
    }
}

Exposure mk_exposure(const ScenarioSchema& sc, int salt, int64_t ts) {
    Exposure e;
    e.scenario_id = sc.scenario_id;
    for (size_t k = 0; k < sc.user_feature_vocabs.size(); ++k) e.user_features.push_back((salt + 3 * static_cast<int>(k)) % sc.user_feature_vocabs[k]);
    for (size_t k = 0; k < sc.cross_feature_vocabs.size(); ++k) e.cross_features.push_back((salt * 7 + static_cast<int>(k)) % sc.cross_feature_vocabs[k]);
    for (size_t k = 0; k < sc.item_feature_vocabs.size(); ++k) e.item_features.push_back((salt * 13 + 5 * static_cast<int>(k)) % sc.item_feature_vocabs[k]);
    e.timestamp = ts;
    return e;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << "usage: ref_agg OUT\n";
        return 2;
    }
    try {
        mtfa::Writer w(argv[1]);
        GeneratorConfig gc;
        gc.n_scenarios = 4;
        gc.n_users = 64;
        gc.seq_len_min = 0;
        gc.seq_len_max = 21;
        gc.exposures_min = 0;
        gc.exposures_max = 6;
        gc.seed = 21;
        Dataset d = generate_dataset(gc);
        int k = 0;
        {
            // 0: the dataset's exposures re-streamed in a seeded shuffle; store = every user,
            // plus users that have no exposures (not emitted by aggregate_users)
            Stream st;
            std::map<int64_t, UserContext> store;
            for (const auto& s : d.samples) {
                store[s.user_id] = UserContext{s.historical_sequences, s.realtime_sequences};
                for (const auto& e : s.exposures) st.pairs.emplace_back(s.user_id, e);
            }
            for (int u = 0; u < 5; ++u) store[100000 + 7 * u] = UserContext{d.samples[u].historical_sequences, {}};
            Rng rng(77);
            for (size_t i = st.pairs.size(); i > 1; --i) std::swap(st.pairs[i - 1], st.pairs[rng.next_below(i)]);
            run_case(w, k++, d, st, store);
        }
        const ScenarioSchema& s0 = d.scenario(0);
        const ScenarioSchema& s1 = d.scenario(1);
        {
            // 1: test_schema_data.cpp:122-131 — one user, 2 exposures in scenario 1 then 3 in 0, interleaved
            Stream st;
            std::map<int64_t, UserContext> store;
            store[42] = {};
            int salt = 0;
            for (int i = 0; i < 5; ++i) st.pairs.emplace_back(42, mk_exposure(i % 2 ? s1 : s0, salt++, 1500 - i));
            run_case(w, k++, d, st, store);
        }
        {
            // 2: test_schema_data.cpp:133-141 — 100 users x 8 exposures, users streamed in descending order
            Stream st;
            std::map<int64_t, UserContext> store;
            for (int64_t u = 0; u < 100; ++u) store[u] = {d.samples[u % d.samples.size()].historical_sequences,
                                                          d.samples[u % d.samples.size()].realtime_sequences};
            for (int i = 0; i < 8; ++i)
                for (int64_t u = 99; u >= 0; --u) st.pairs.emplace_back(u, mk_exposure(i % 2 ? s1 : s0, static_cast<int>(u * 8 + i), 1000 + i));
            run_case(w, k++, d, st, store);
        }
        {
            // 3: unknown user at index 3 before an unknown scenario at index 5 -> "unknown user"
            Stream st;
            std::map<int64_t, UserContext> store;
            store[5] = {};
            store[9] = {};
            for (int i = 0; i < 7; ++i) {
                Exposure e = mk_exposure(s0, i, 1000 + i);
                int64_t u = i % 2 ? 5 : 9;
                if (i == 3) u = 6;
                if (i == 5) e.scenario_id = 77;
                st.pairs.emplace_back(u, e);
            }
            run_case(w, k++, d, st, store);
        }
        {
            // 4: unknown scenario at index 2 before an unknown user at index 4 -> "unknown scenario 77";
            // index 6 carries both faults (scenario checked first)
            Stream st;
            std::map<int64_t, UserContext> store;
            store[5] = {};
            for (int i = 0; i < 8; ++i) {
                Exposure e = mk_exposure(s1, i, 1000 + i);
                int64_t u = 5;
                if (i == 2) e.scenario_id = 77;
                if (i == 4) u = 8;
                if (i == 6) {
                    e.scenario_id = 99;
                    u = 11;
                }
                st.pairs.emplace_back(u, e);
            }
            run_case(w, k++, d, st, store);
        }
        {
            // 5: empty stream
            Stream st;
            std::map<int64_t, UserContext> store;
            store[3] = {d.samples[0].historical_sequences, d.samples[0].realtime_sequences};
            run_case(w, k++, d, st, store);
        }
        w.put("n_cases", std::vector<int32_t>{k});
        std::cerr << "ref_agg: " << k << " cases -> " << argv[1] << "\n";
    } catch (const std::exception& e) {
        std::cerr << "ref_agg: " << e.what() << "\n";
        return 1;
    }
    return 0;
}
