// ref_dump.cpp — golden-vector generator built from the UNMODIFIED reference
// sources under /root/reference/proj (compiled by oracle/Makefile into
// oracle/_ref/ref_dump).
//
// TEST INFRASTRUCTURE ONLY: this program exists to pin the numpy restatement
// (oracle/mtfm_oracle.py) and the CUDA path against the reference itself. It
// calls only public reference entry points:
//   generate_dataset            proj/src/datagen.cpp:218
//   Model<Real>::build           proj/include/mtfm/model.hpp:126
//   plan_tokens                  proj/include/mtfm/tokenizer.hpp:53
//   assemble_tokens              proj/include/mtfm/tokenizer.hpp:240
//   Model::make_geom             proj/include/mtfm/model.hpp:360
//   target/full_attention_layer  proj/include/mtfm/hta.hpp:138,158
//   mmoe_forward                 proj/include/mtfm/heads.hpp:47
//   Model::forward_sample        proj/include/mtfm/model.hpp:251 (cross-check)
// and writes an MTFA archive (oracle/mtfa.hpp) with the dataset in the packed
// jagged layout of include/mtfm_cuda.h, the model config, parameter
// checksums (optionally full parameters), the token plan, per-layer
// activations and the per-record logits/probabilities in f64 and f32.
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <string>
#include <vector>

#include "jitter.hpp"
#include "mtfa.hpp"
#include "mtfm/datagen.hpp"
#include "mtfm/model.hpp"
#include "mtfm/prune.hpp"
#include "mtfm/train.hpp"
#include "mtfm/verify.hpp"

using namespace mtfm;

namespace {

struct Opts {
    std::string out;
    std::string preset = "gen";  // gen | micro
    GeneratorConfig gc;
    ModelConfig mc;
    uint64_t model_seed = 7;
    int hlen = -1, rlen = -1;  // fixed lengths by order-preserving subsample
    int dump_x_users = 0;      // users whose per-layer activations are dumped
    bool params = false;       // dump full f32 parameters
    uint64_t jitter = 0;       // != 0: perturb biases / GLN affines / towers (jitter_params)
    double tower_scale = 1.0;
    int train_steps = 0;       // > 0: Trainer::train_step over every user of the batch, dumped
    bool prune = false;        // prune_model_projections (prune.hpp:92-103) before the forwards
    double lr = 1e-3;
};

Opts parse(int argc, char** argv) {
    Opts o;
    o.gc.n_scenarios = 4;
    o.gc.n_users = 8;
    o.gc.n_hist_seqs = 2;
    o.gc.n_rt_seqs = 1;
    o.gc.seq_len_min = 0;
    o.gc.seq_len_max = 21;
    o.gc.exposures_min = 0;
    o.gc.exposures_max = 2;
    o.gc.seed = 1;
    o.mc.hta.d_model = 64;
    o.mc.hta.blocks = 1;
    o.mc.hta.target_layers = 1;
    o.mc.hta.full_layers = 1;
    o.mc.hta.heads = 4;
    o.mc.hta.kv_heads = 2;
    o.mc.d_emb = 16;
    o.mc.experts = 4;
    o.mc.d_expert = 64;
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        auto nxt = [&]() -> std::string {
            if (i + 1 >= argc) throw config_error("missing value for " + a);
            return argv[++i];
        };
        if (a == "--out") o.out = nxt();
        else if (a == "--preset") o.preset = nxt();
        else if (a == "--users") o.gc.n_users = std::stoi(nxt());
        else if (a == "--scen") o.gc.n_scenarios = std::stoi(nxt());
        else if (a == "--nh") o.gc.n_hist_seqs = std::stoi(nxt());
        else if (a == "--nr") o.gc.n_rt_seqs = std::stoi(nxt());
        else if (a == "--lenmin") o.gc.seq_len_min = std::stoi(nxt());
        else if (a == "--lenmax") o.gc.seq_len_max = std::stoi(nxt());
        else if (a == "--expmin") o.gc.exposures_min = std::stoi(nxt());
        else if (a == "--expmax") o.gc.exposures_max = std::stoi(nxt());
        else if (a == "--gseed") o.gc.seed = std::stoull(nxt());
        else if (a == "--d") o.mc.hta.d_model = std::stoi(nxt());
        else if (a == "--blocks") o.mc.hta.blocks = std::stoi(nxt());
        else if (a == "--K") o.mc.hta.target_layers = std::stoi(nxt());
        else if (a == "--P") o.mc.hta.full_layers = std::stoi(nxt());
        else if (a == "--H") o.mc.hta.heads = std::stoi(nxt());
        else if (a == "--G") o.mc.hta.kv_heads = std::stoi(nxt());
        else if (a == "--norm") o.mc.hta.norm = attn_norm_from_string(nxt());
        else if (a == "--demb") o.mc.d_emb = std::stoi(nxt());
        else if (a == "--E") o.mc.experts = std::stoi(nxt());
        else if (a == "--dexp") o.mc.d_expert = std::stoi(nxt());
        else if (a == "--mseed") o.model_seed = std::stoull(nxt());
        else if (a == "--hlen") o.hlen = std::stoi(nxt());
        else if (a == "--rlen") o.rlen = std::stoi(nxt());
        else if (a == "--dumpx") o.dump_x_users = std::stoi(nxt());
        else if (a == "--params") o.params = true;
        else if (a == "--jitter") o.jitter = std::stoull(nxt());
        else if (a == "--tower-scale") o.tower_scale = std::stod(nxt());
        else if (a == "--train") o.train_steps = std::stoi(nxt());
        else if (a == "--prune") o.prune = true;
        else if (a == "--lr") o.lr = std::stod(nxt());
        else throw config_error("unknown flag " + a);
    }
    if (o.out.empty()) throw config_error("--out required");
    return o;
}

// Seeded order-preserving subsample of a sequence down to `len` events.
void subsample(SequenceRecord& rec, int len, Rng& rng) {
    if (len < 0 || static_cast<int>(rec.events.size()) <= len) return;
    std::vector<int> keep(rec.events.size());
    for (size_t i = 0; i < keep.size(); ++i) keep[i] = static_cast<int>(i);
    // partial Fisher-Yates, then restore order
    for (int i = 0; i < len; ++i) {
        int j = i + static_cast<int>(rng.next_below(keep.size() - static_cast<size_t>(i)));
        std::swap(keep[static_cast<size_t>(i)], keep[static_cast<size_t>(j)]);
    }
    keep.resize(static_cast<size_t>(len));
    std::sort(keep.begin(), keep.end());
    std::vector<BehaviorEvent> ev;
    for (int k : keep) ev.push_back(rec.events[static_cast<size_t>(k)]);
    rec.events = std::move(ev);
}

struct Packed {
    std::vector<int64_t> user_id;
    std::vector<int32_t> seq_off{0}, seq_schema, ev_off{0}, ev_feat_off{0}, ev_feats;
    std::vector<uint8_t> seq_kind;
    std::vector<int64_t> ev_ts;
    std::vector<int32_t> exp_off{0}, exp_scenario, exp_feat_off{0}, exp_blk, exp_feats, exp_labels;
    std::vector<int64_t> exp_ts;
};

void pack(const SchemaSet& ss, const std::vector<UserSample>& samples, Packed& p, int max_tasks) {
    for (const auto& s : samples) {
        p.user_id.push_back(s.user_id);
        auto eat = [&](const std::vector<SequenceRecord>& seqs, uint8_t kind) {
            for (const auto& rec : seqs) {
                p.seq_kind.push_back(kind);
                p.seq_schema.push_back(rec.seq_schema_id);
                for (const auto& ev : rec.events) {
                    p.ev_ts.push_back(ev.timestamp);
                    for (int f : ev.item_features) p.ev_feats.push_back(f);
                    p.ev_feat_off.push_back(static_cast<int32_t>(p.ev_feats.size()));
                }
                p.ev_off.push_back(static_cast<int32_t>(p.ev_ts.size()));
            }
        };
        eat(s.historical_sequences, 0);
        eat(s.realtime_sequences, 1);
        p.seq_off.push_back(static_cast<int32_t>(p.seq_kind.size()));
        for (const auto& e : s.exposures) {
            p.exp_scenario.push_back(e.scenario_id);
            p.exp_ts.push_back(e.timestamp);
            p.exp_blk.push_back(static_cast<int32_t>(e.user_features.size()));
            p.exp_blk.push_back(static_cast<int32_t>(e.cross_features.size()));
            p.exp_blk.push_back(static_cast<int32_t>(e.item_features.size()));
            for (int f : e.user_features) p.exp_feats.push_back(f);
            for (int f : e.cross_features) p.exp_feats.push_back(f);
            for (int f : e.item_features) p.exp_feats.push_back(f);
            p.exp_feat_off.push_back(static_cast<int32_t>(p.exp_feats.size()));
            std::vector<int32_t> lab(static_cast<size_t>(max_tasks), -1);
            try {
                const auto& sc = ss.scenario(e.scenario_id);
                for (size_t t = 0; t < sc.tasks.size(); ++t) {
                    auto it = e.labels.find(sc.tasks[t]);
                    if (it != e.labels.end()) lab[t] = it->second;
                }
            } catch (const integrity_error&) {
            }
            for (auto v : lab) p.exp_labels.push_back(v);
        }
        p.exp_off.push_back(static_cast<int32_t>(p.exp_scenario.size()));
    }
}

void put_schemas(mtfa::Writer& w, const SchemaSet& ss) {
    auto seqs = [&](const std::string& key, const std::vector<SequenceSchema>& v) {
        std::vector<int32_t> ids, nslots, vocabs;
        for (const auto& s : v) {
            ids.push_back(s.seq_id);
            nslots.push_back(static_cast<int32_t>(s.feature_vocabs.size()));
            for (int x : s.feature_vocabs) vocabs.push_back(x);
        }
        w.put("schema/" + key + "/ids", ids);
        w.put("schema/" + key + "/nslots", nslots);
        w.put("schema/" + key + "/vocabs", vocabs);
    };
    seqs("hist", ss.hist);
    seqs("rt", ss.rt);
    std::vector<int32_t> ids, nu, nc, ni, vocabs;
    std::string tasks;
    for (const auto& s : ss.scenarios) {
        ids.push_back(s.scenario_id);
        nu.push_back(static_cast<int32_t>(s.user_feature_vocabs.size()));
        nc.push_back(static_cast<int32_t>(s.cross_feature_vocabs.size()));
        ni.push_back(static_cast<int32_t>(s.item_feature_vocabs.size()));
        for (int x : s.user_feature_vocabs) vocabs.push_back(x);
        for (int x : s.cross_feature_vocabs) vocabs.push_back(x);
        for (int x : s.item_feature_vocabs) vocabs.push_back(x);
        for (size_t t = 0; t < s.tasks.size(); ++t) tasks += (t ? "," : "") + s.tasks[t];
        tasks += ";";
    }
    w.put("schema/scen/ids", ids);
    w.put("schema/scen/nu", nu);
    w.put("schema/scen/nc", nc);
    w.put("schema/scen/ni", ni);
    w.put("schema/scen/vocabs", vocabs);
    w.put_str("schema/scen/tasks", tasks);
}

}  // namespace

int main(int argc, char** argv) {
    try {
        Opts o = parse(argc, argv);
        SchemaSet ss;
        std::vector<UserSample> samples;
        if (o.preset == "micro") {
            ss = micro_schemas();
            o.mc = micro_model_config();
            o.model_seed = 5;
            samples = {micro_sample()};
        } else {
            Dataset d = generate_dataset(o.gc);
            ss = SchemaSet::from(d);
            samples = d.samples;
            for (auto& s : samples) {
                Rng rng(o.gc.seed * 7919ULL + 1000ULL + static_cast<uint64_t>(s.user_id));
                for (auto& rec : s.historical_sequences) subsample(rec, o.hlen, rng);
                for (auto& rec : s.realtime_sequences) subsample(rec, o.rlen, rng);
            }
        }

        Model<float> m32 = Model<float>::build(ss, o.mc, o.model_seed);
        if (o.jitter) jitter_params(m32.params, o.jitter, o.tower_scale);
        PruneReport prep;
        if (o.prune) prep = prune_model_projections(m32.params);
        Model<double> m64 = Model<double>::build(ss, o.mc, o.model_seed);
        // The f64 model carries exactly the f32 weights, so it is the exact
        // answer for the weights the GPU path receives.
        for (auto& e : m64.params) {
            const auto& src = m32.params.at(e.name).value;
            for (size_t i = 0; i < e.value.size(); ++i) e.value[i] = static_cast<double>(src[i]);
        }

        mtfa::Writer w(o.out);
        put_schemas(w, ss);
        const HTAConfig& h = o.mc.hta;
        w.put("config/ints", std::vector<int32_t>{h.d_model, h.blocks, h.target_layers, h.full_layers,
                                                  h.heads, h.kv_heads, static_cast<int32_t>(h.norm),
                                                  o.mc.d_emb, o.mc.experts, o.mc.d_expert});
        w.put("config/eps", std::vector<double>{h.eps});
        w.put("config/model_seed", std::vector<int64_t>{static_cast<int64_t>(o.model_seed)});
        w.put("config/jitter", std::vector<double>{static_cast<double>(o.jitter), o.tower_scale});
        if (o.prune) {
            w.put("prune/report", std::vector<int64_t>{static_cast<int64_t>(prep.groups_covered),
                                                      static_cast<int64_t>(prep.zeros_written),
                                                      static_cast<int64_t>(prep.exempt_tail_rows),
                                                      static_cast<int64_t>(prep.pruned_params.size())});
            for (const auto& n : prep.pruned_params) {
                const auto& t = m32.params.at(n).value;
                std::vector<float> v(t.size());
                for (size_t i = 0; i < v.size(); ++i) v[i] = t[i];
                w.put("prune/param/" + n, v, {static_cast<int64_t>(t.rows()), static_cast<int64_t>(t.cols())});
            }
        }

        int max_tasks = 0;
        for (const auto& s : ss.scenarios) max_tasks = std::max(max_tasks, static_cast<int>(s.tasks.size()));
        Packed p;
        pack(ss, samples, p, max_tasks);
        w.put("batch/user_id", p.user_id);
        w.put("batch/seq_off", p.seq_off);
        w.put("batch/seq_kind", p.seq_kind);
        w.put("batch/seq_schema", p.seq_schema);
        w.put("batch/ev_off", p.ev_off);
        w.put("batch/ev_ts", p.ev_ts);
        w.put("batch/ev_feat_off", p.ev_feat_off);
        w.put("batch/ev_feats", p.ev_feats);
        w.put("batch/exp_off", p.exp_off);
        w.put("batch/exp_scenario", p.exp_scenario);
        w.put("batch/exp_ts", p.exp_ts);
        w.put("batch/exp_feat_off", p.exp_feat_off);
        w.put("batch/exp_blk", p.exp_blk);
        w.put("batch/exp_feats", p.exp_feats);
        w.put("batch/exp_labels", p.exp_labels,
              {static_cast<int64_t>(p.exp_scenario.size()), static_cast<int64_t>(max_tasks)});

        // Parameters: names in registration order plus checksums (and values).
        std::string names;
        std::vector<double> sums, sqs;
        std::vector<int64_t> shapes;
        for (const auto& e : m32.params) {
            names += e.name + "\n";
            double s = 0, q = 0;
            for (size_t i = 0; i < e.value.size(); ++i) {
                s += e.value[i];
                q += static_cast<double>(e.value[i]) * e.value[i];
            }
            sums.push_back(s);
            sqs.push_back(q);
            shapes.push_back(static_cast<int64_t>(e.value.rows()));
            shapes.push_back(static_cast<int64_t>(e.value.cols()));
            if (o.params) {
                std::vector<float> v(e.value.size());
                for (size_t i = 0; i < v.size(); ++i) v[i] = e.value[i];
                w.put("param/" + e.name, v,
                      {static_cast<int64_t>(e.value.rows()), static_cast<int64_t>(e.value.cols())});
            }
        }
        w.put_str("params/names", names);
        w.put("params/sum", sums);
        w.put("params/sumsq", sqs);
        w.put("params/shape", shapes, {static_cast<int64_t>(sums.size()), 2});

        // Plan + forward per user.
        std::vector<int32_t> plan_off{0}, meta_group, meta_exp, f2p, tok_group, valid, bounds;
        std::vector<uint8_t> meta_kind;
        std::vector<int64_t> meta_ts;
        std::vector<int32_t> xoff{0};
        std::vector<double> x0s, xlayers;
        std::vector<int64_t> rec_user;
        std::vector<int32_t> rec_scen, rec_exp, rec_task, rec_label;
        std::vector<double> prob64, prob32, logit64;
        std::vector<float> logit32;
        const int n_layers = h.blocks * h.layers_per_block();
        size_t dumped = 0;

        for (size_t ui = 0; ui < samples.size(); ++ui) {
            const UserSample& s = samples[ui];
            TokenPlan plan = plan_tokens(s);
            std::vector<int> groups;
            for (const auto& m : plan.metas) groups.push_back(m32.groups.group_of(m));
            MaskMatrix mask = build_mask(plan.metas);
            auto counts = mask.row_valid_counts();
            for (size_t i = 0; i < plan.metas.size(); ++i) {
                meta_kind.push_back(static_cast<uint8_t>(plan.metas[i].kind));
                meta_group.push_back(plan.metas[i].group_id);
                meta_ts.push_back(plan.metas[i].timestamp);
                meta_exp.push_back(plan.metas[i].exposure_ref);
                f2p.push_back(plan.final_to_pile[i]);
                tok_group.push_back(groups[i]);
                valid.push_back(counts[i]);
            }
            plan_off.push_back(static_cast<int32_t>(meta_kind.size()));
            bounds.push_back(plan.bounds.l_h);
            bounds.push_back(plan.bounds.l_r);
            bounds.push_back(plan.bounds.l_t);

            // f64 forward, layer by layer through the public layer functions.
            auto run = [&](auto& model, auto tag, bool dump) {
                using M = std::remove_reference_t<decltype(model)>;
                using Real = std::remove_reference_t<decltype(model.params.at(0).value[0])>;
                (void)tag;
                using Ctx = EvalCtx<std::remove_const_t<Real>>;
                Ctx ctx;
                auto refs = model.bind_eval(model.params);
                auto x = assemble_tokens(ctx, s, plan, refs.tok);
                auto geom = model.make_geom(plan);
                if (dump)
                    for (size_t i = 0; i < ctx.val(x).size(); ++i) x0s.push_back(ctx.val(x)[i]);
                size_t li = 0;
                for (int b = 0; b < h.blocks; ++b) {
                    for (int k = 0; k < h.layers_per_block(); ++k, ++li) {
                        if (k < h.target_layers)
                            x = target_attention_layer(ctx, x, refs.stack.layers[li], geom);
                        else
                            x = full_attention_layer(ctx, x, refs.stack.layers[li], geom);
                        if (dump)
                            for (size_t i = 0; i < ctx.val(x).size(); ++i) xlayers.push_back(ctx.val(x)[i]);
                    }
                }
                const size_t off = static_cast<size_t>(plan.bounds.l_h + plan.bounds.l_r);
                auto t_rows = ctx.slice_rows(x, off, static_cast<size_t>(plan.bounds.total()));
                std::vector<TokenMeta> t_metas(plan.metas.begin() + static_cast<long>(off), plan.metas.end());
                auto logits = mmoe_forward(ctx, t_rows, t_metas, model.schemas.tasks_by_scenario(), refs.heads);
                (void)sizeof(M);
                return logits;
            };
            const bool dump = dumped < static_cast<size_t>(o.dump_x_users);
            auto l64 = run(m64, 0, dump);
            if (dump) {
                ++dumped;
                xoff.push_back(static_cast<int32_t>(x0s.size() / static_cast<size_t>(h.d_model)));
            }
            auto l32 = run(m32, 0, false);
            auto r64 = m64.forward_sample(s);
            auto r32 = m32.forward_sample(s);
            size_t ri = 0;
            for (size_t c = 0; c < l64.columns.size(); ++c) {
                const auto& col = l64.columns[c];
                const auto& z64 = *col.logits;
                const auto& z32 = *l32.columns[c].logits;
                const auto& sc = ss.scenario(col.scenario_id);
                int task_idx = -1;
                for (size_t t = 0; t < sc.tasks.size(); ++t)
                    if (sc.tasks[t] == col.task) task_idx = static_cast<int>(t);
                for (size_t i = 0; i < z64.rows(); ++i, ++ri) {
                    const auto& a = r64.at(ri);
                    const auto& b = r32.at(ri);
                    if (a.exposure_index != col.exposure_refs[i] || a.task != col.task ||
                        b.exposure_index != a.exposure_index)
                        throw contract_error("record order cross-check failed");
                    rec_user.push_back(s.user_id);
                    rec_scen.push_back(col.scenario_id);
                    rec_exp.push_back(col.exposure_refs[i]);
                    rec_task.push_back(task_idx);
                    rec_label.push_back(a.label);
                    prob64.push_back(a.probability);
                    prob32.push_back(b.probability);
                    logit64.push_back(z64.at(i, 0));
                    logit32.push_back(z32.at(i, 0));
                }
            }
            if (ri != r64.size()) throw contract_error("record count cross-check failed");
        }
        w.put("plan/off", plan_off);
        w.put("plan/kind", meta_kind);
        w.put("plan/group_id", meta_group);
        w.put("plan/ts", meta_ts);
        w.put("plan/exposure_ref", meta_exp);
        w.put("plan/final_to_pile", f2p);
        w.put("plan/token_group", tok_group);
        w.put("plan/valid_count", valid);
        w.put("plan/bounds", bounds, {static_cast<int64_t>(samples.size()), 3});
        const int64_t dm = h.d_model;
        w.put("fwd/x_off", xoff);
        w.put("fwd/x0", x0s, {static_cast<int64_t>(x0s.size()) / dm, dm});
        // user-major, then layer-major: user u contributes n_layers * N_u rows.
        w.put("fwd/x_layers", xlayers, {static_cast<int64_t>(xlayers.size()) / dm, dm});
        w.put("fwd/n_layers", std::vector<int32_t>{n_layers});
        w.put("rec/user", rec_user);
        w.put("rec/scenario", rec_scen);
        w.put("rec/exposure", rec_exp);
        w.put("rec/task", rec_task);
        w.put("rec/label", rec_label);
        w.put("rec/prob64", prob64);
        w.put("rec/prob32", prob32);
        w.put("rec/logit64", logit64);
        w.put("rec/logit32", logit32);
        if (o.train_steps > 0) {
            // Trainer::train_step (train.hpp:111-147) on the f64 model carrying the f32 weights:
            // every user of the batch in one minibatch, one worker; the per-parameter gradients
            // of step 1 (already x 1/batch, before clipping), the parameters after step 1 and
            // after the last step, and the per-step losses
            Model<double> mt = m64;
            Dataset dd;
            dd.hist_seq_schemas = ss.hist;
            dd.rt_seq_schemas = ss.rt;
            dd.scenarios = ss.scenarios;
            dd.samples = samples;
            TrainConfig tc;
            tc.batch_size = static_cast<int>(samples.size());
            tc.threads = 1;
            tc.adam.lr = o.lr;
            Trainer<double> tr(mt, dd, tc);
            std::vector<const UserSample*> batch;
            for (const auto& s : dd.samples) batch.push_back(&s);
            std::vector<double> losses;
            for (int step = 0; step < o.train_steps; ++step) {
                losses.push_back(tr.train_step(batch));
                if (step == 0)
                    for (const auto& e : mt.params) {
                        std::vector<float> g(e.grad.size()), v(e.value.size());
                        for (size_t i = 0; i < g.size(); ++i) g[i] = static_cast<float>(e.grad[i]);
                        for (size_t i = 0; i < v.size(); ++i) v[i] = static_cast<float>(e.value[i]);
                        const std::vector<int64_t> sh{static_cast<int64_t>(e.value.rows()), static_cast<int64_t>(e.value.cols())};
                        w.put("train/grad/" + e.name, g, sh);
                        w.put("train/param1/" + e.name, v, sh);
                    }
            }
            for (const auto& e : mt.params) {
                std::vector<float> v(e.value.size());
                for (size_t i = 0; i < v.size(); ++i) v[i] = static_cast<float>(e.value[i]);
                w.put("train/paramN/" + e.name, v,
                      {static_cast<int64_t>(e.value.rows()), static_cast<int64_t>(e.value.cols())});
            }
            w.put("train/loss", losses);
            w.put("train/cfg", std::vector<double>{o.lr, tc.adam.beta1, tc.adam.beta2, tc.adam.eps, tc.adam.clip_norm,
                                                   static_cast<double>(o.train_steps)});
        }
        std::cerr << "ref_dump: " << samples.size() << " users, " << rec_user.size() << " records -> "
                  << o.out << "\n";
    } catch (const std::exception& e) {
        std::cerr << "ref_dump: " << e.what() << "\n";
        return 1;
    }
    return 0;
}
