// ref_integration.cpp — drop-in check: the reference's own model, data and
// forward_sample (CPU) against include/mtfm_cuda.hpp (GPU) in one process.
//
// TEST INFRASTRUCTURE ONLY (built by oracle/Makefile into oracle/_ref/, linked
// against the unmodified reference sources and libmtfm_cuda.so). Checks, for
// a generated dataset: identical record keys and labels, max |dp| and max
// |dlogit| of GpuModel::forward_samples vs Model<float>::forward_sample
// (model.hpp:251), GpuModel::infer_request vs infer_request (subgraph.hpp:47),
// and that an out-of-vocab id surfaces as mtfm::lookup_error.
// Prints one JSON line; exit code 0 iff every check passes.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "jitter.hpp"
#include "mtfm/datagen.hpp"
#include "mtfm/model.hpp"
#include "mtfm/subgraph.hpp"
#include "mtfm_cuda.hpp"

using namespace mtfm;

static double logit(double p) { return std::log(p / (1.0 - p)); }

int main(int argc, char** argv) {
    int precision = MTFM_PRECISION_BF16;
    int users = 16;
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        if (a == "--fp32") precision = MTFM_PRECISION_FP32_CHECK;
        if (a == "--users" && i + 1 < argc) users = std::stoi(argv[++i]);
    }
    GeneratorConfig gc;
    gc.n_scenarios = 4;
    gc.n_users = users;
    gc.n_hist_seqs = 2;
    gc.n_rt_seqs = 1;
    gc.seq_len_min = 8;
    gc.seq_len_max = 96;
    gc.exposures_min = 0;
    gc.exposures_max = 6;
    gc.seed = 17;
    Dataset d = generate_dataset(gc);
    ModelConfig mc;
    mc.hta.d_model = 128;
    mc.hta.blocks = 2;
    mc.hta.target_layers = 3;
    mc.hta.full_layers = 1;
    mc.hta.heads = 4;
    mc.hta.kv_heads = 2;
    mc.d_expert = 128;
    Model<float> model = Model<float>::build(SchemaSet::from(d), mc, 7);
    // off the default init: every bias and GLN gain/bias (jitter.hpp), towers unscaled so the
    // bf16 logit tolerance (2e-2 absolute) is not dominated by bf16 storage error
    jitter_params(model.params, 201, 1.0);

    bool ok = true;
    double max_dp = 0, max_dz = 0;
    size_t n_rec = 0;
    try {
        cuda::GpuModel gpu(model, 0, precision);
        std::vector<PredictionRecord> want;
        for (const auto& s : d.samples) {
            auto r = model.forward_sample(s);
            want.insert(want.end(), r.begin(), r.end());
        }
        auto got = gpu.forward_samples(d.samples);
        n_rec = want.size();
        if (got.size() != want.size()) ok = false;
        for (size_t i = 0; ok && i < want.size(); ++i) {
            const auto& a = want[i];
            const auto& b = got[i];
            if (a.user_id != b.user_id || a.scenario_id != b.scenario_id || a.exposure_index != b.exposure_index ||
                a.task != b.task || a.label != b.label)
                ok = false;
            max_dp = std::max(max_dp, std::fabs(a.probability - b.probability));
            max_dz = std::max(max_dz, std::fabs(logit(a.probability) - logit(b.probability)));
        }
        const double tol = precision == MTFM_PRECISION_BF16 ? 2e-2 : 1e-4;
        if (max_dz > tol) ok = false;

        // request-level serving path vs the reference's subgraph inference
        auto sub = extract_subgraph(model, 1);
        InferenceRequest req;
        req.user_id = d.samples[0].user_id;
        req.scenario_id = 1;
        req.timestamp = 1500;
        req.historical_sequences = d.samples[0].historical_sequences;
        req.realtime_sequences = d.samples[0].realtime_sequences;
        const auto& sc = d.scenario(1);
        for (int c = 0; c < 5; ++c) {
            Candidate cand;
            for (size_t k = 0; k < sc.user_feature_vocabs.size(); ++k) cand.user_features.push_back((c * 7 + 3) % sc.user_feature_vocabs[k]);
            for (size_t k = 0; k < sc.cross_feature_vocabs.size(); ++k) cand.cross_features.push_back((c * 5 + 1) % sc.cross_feature_vocabs[k]);
            for (size_t k = 0; k < sc.item_feature_vocabs.size(); ++k) cand.item_features.push_back((c * 11 + 2) % sc.item_feature_vocabs[k]);
            req.candidates.push_back(cand);
        }
        auto rw = infer_request(model, sub, req);
        auto rg = gpu.infer_request(req);
        if (rw.size() != rg.size()) ok = false;
        for (size_t i = 0; ok && i < rw.size(); ++i) {
            if (rw[i].exposure_index != rg[i].exposure_index || rw[i].task != rg[i].task) ok = false;
            if (std::fabs(logit(rw[i].probability) - logit(rg[i].probability)) > tol) ok = false;
        }

        // scenario deployment: only extract_subgraph(model, 1)'s ParamStore uploaded, and
        // many requests in one forward == one infer_request each (subgraph.hpp:47-62)
        cuda::GpuModel gsub(sub, 0, precision);
        std::vector<InferenceRequest> reqs;
        for (size_t u = 0; u < d.samples.size() && reqs.size() < 12; u += 2) {
            InferenceRequest q = req;
            q.user_id = d.samples[u].user_id;
            q.timestamp = 1200 + static_cast<int64_t>(u);
            q.historical_sequences = d.samples[u].historical_sequences;
            q.realtime_sequences = d.samples[u].realtime_sequences;
            q.candidates.resize(1 + u % 4, req.candidates[u % req.candidates.size()]);
            reqs.push_back(q);
        }
        auto batched = gsub.infer_requests(reqs);
        for (size_t i = 0; ok && i < reqs.size(); ++i) {
            auto want1 = infer_request(model, sub, reqs[i]);
            auto alone = gsub.infer_request(reqs[i]);
            if (batched[i].size() != want1.size() || alone.size() != want1.size()) ok = false;
            for (size_t j = 0; ok && j < want1.size(); ++j) {
                if (batched[i][j].exposure_index != want1[j].exposure_index || batched[i][j].task != want1[j].task ||
                    batched[i][j].user_id != want1[j].user_id)
                    ok = false;
                if (batched[i][j].probability != alone[j].probability) ok = false;  // batching is bitwise neutral
                if (std::fabs(logit(batched[i][j].probability) - logit(want1[j].probability)) > tol) ok = false;
            }
        }
        // a subgraph refuses another scenario's request (subgraph.hpp:51-55)
        {
            InferenceRequest other = req;
            other.scenario_id = 2;
            bool threw = false;
            try {
                gsub.infer_request(other);
            } catch (const integrity_error&) {
                threw = true;
            }
            if (!threw) ok = false;
        }
        if (!ok) std::printf("{\"stage\": \"subgraph\"}\n");

        // error taxonomy: out-of-vocab id -> lookup_error (eval_ctx.hpp:193-194)
        UserSample bad = d.samples[0];
        bad.exposures.at(0).item_features.at(0) = 1 << 20;
        bool threw = false;
        try {
            gpu.forward_sample(bad);
        } catch (const lookup_error&) {
            threw = true;
        }
        if (!threw) ok = false;
    } catch (const std::exception& e) {
        std::printf("{\"ok\": false, \"error\": \"%s\"}\n", e.what());
        return 1;
    }
    std::printf("{\"ok\": %s, \"precision\": \"%s\", \"users\": %zu, \"records\": %zu, \"max_abs_dp\": %.3e, "
                "\"max_abs_dlogit\": %.3e}\n",
                ok ? "true" : "false", precision == MTFM_PRECISION_BF16 ? "bf16" : "fp32", d.samples.size(), n_rec,
                max_dp, max_dz);
    return ok ? 0 : 1;
}
