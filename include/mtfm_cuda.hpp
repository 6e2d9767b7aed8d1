// mtfm_cuda.hpp — C++ drop-in shim: the reference model API on top of the
// C ABI of mtfm_cuda.h (libmtfm_cuda.so).
//
// Header-only; include it after the reference headers (it uses the
// reference's own types, /root/reference/proj/include/mtfm):
//
//   #include "mtfm/model.hpp"      // Model<Real>, UserSample, PredictionRecord, ...
//   #include "mtfm_cuda.hpp"
//
//   mtfm::Model<float> model = ...;                  // built / loaded as before
//   mtfm::cuda::GpuModel gpu(model);                 // uploads ParamStore by name
//   auto recs = gpu.forward_samples(samples);        // == concatenated model.forward_sample(s)
//   auto one  = gpu.forward_sample(sample);          // == model.forward_sample(sample)
//   auto req  = gpu.infer_request(request);          // == infer_request(model, subgraph, request)
//
// Replaces (paths relative to /root/reference/proj):
//   Model<Real>::forward_sample / forward_with / forward_scoped   model.hpp:244-312
//   infer_request                                                  subgraph.hpp:47-62
// Errors are rethrown as the reference exception types (errors.hpp:9-40), with
// the message of the device-side check; CUDA failures throw std::runtime_error.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "mtfm_cuda.h"

namespace mtfm {
namespace cuda {

[[noreturn]] inline void rethrow(mtfm_status s) {
    const std::string msg = mtfm_cuda_last_error();
    switch (s) {
        case MTFM_CONFIG_ERROR: throw config_error(msg);
        case MTFM_INTEGRITY_ERROR: throw integrity_error(msg);
        case MTFM_DIMENSION_ERROR: throw dimension_error(msg);
        case MTFM_PARSE_ERROR: throw parse_error(msg);
        case MTFM_LOOKUP_ERROR: throw lookup_error(msg);
        case MTFM_CONTRACT_ERROR: throw contract_error(msg);
        default: throw std::runtime_error("mtfm_cuda: " + msg);
    }
}

inline void check(mtfm_status s) {
    if (s != MTFM_OK) rethrow(s);
}

// Packed jagged batch (mtfm_cuda.h layout) built from reference UserSamples.
struct PackedBatch {
    std::vector<int64_t> user_id, ev_ts, exp_ts;
    std::vector<int32_t> seq_off{0}, seq_schema, ev_off{0}, ev_feat_off{0}, ev_feats;
    std::vector<uint8_t> seq_kind;
    std::vector<int32_t> exp_off{0}, exp_scenario, exp_feat_off{0}, exp_blk, exp_feats;

    void add(const UserSample& s) {
        user_id.push_back(s.user_id);
        auto eat = [&](const std::vector<SequenceRecord>& seqs, uint8_t kind) {
            for (const auto& rec : seqs) {
                seq_kind.push_back(kind);
                seq_schema.push_back(rec.seq_schema_id);
                for (const auto& ev : rec.events) {
                    ev_ts.push_back(ev.timestamp);
                    ev_feats.insert(ev_feats.end(), ev.item_features.begin(), ev.item_features.end());
                    ev_feat_off.push_back(static_cast<int32_t>(ev_feats.size()));
                }
                ev_off.push_back(static_cast<int32_t>(ev_ts.size()));
            }
        };
        eat(s.historical_sequences, 0);
        eat(s.realtime_sequences, 1);
        seq_off.push_back(static_cast<int32_t>(seq_kind.size()));
        for (const auto& e : s.exposures) {
            exp_scenario.push_back(e.scenario_id);
            exp_ts.push_back(e.timestamp);
            exp_blk.push_back(static_cast<int32_t>(e.user_features.size()));
            exp_blk.push_back(static_cast<int32_t>(e.cross_features.size()));
            exp_blk.push_back(static_cast<int32_t>(e.item_features.size()));
            exp_feats.insert(exp_feats.end(), e.user_features.begin(), e.user_features.end());
            exp_feats.insert(exp_feats.end(), e.cross_features.begin(), e.cross_features.end());
            exp_feats.insert(exp_feats.end(), e.item_features.begin(), e.item_features.end());
            exp_feat_off.push_back(static_cast<int32_t>(exp_feats.size()));
        }
        exp_off.push_back(static_cast<int32_t>(exp_scenario.size()));
    }

    mtfm_packed_batch view() const {
        mtfm_packed_batch b{};
        b.n_users = static_cast<int32_t>(user_id.size());
        b.n_seqs = static_cast<int32_t>(seq_kind.size());
        b.n_events = static_cast<int32_t>(ev_ts.size());
        b.n_exposures = static_cast<int32_t>(exp_ts.size());
        b.n_ev_feats = static_cast<int64_t>(ev_feats.size());
        b.n_exp_feats = static_cast<int64_t>(exp_feats.size());
        b.user_id = user_id.data();
        b.seq_off = seq_off.data();
        b.seq_kind = seq_kind.data();
        b.seq_schema = seq_schema.data();
        b.ev_off = ev_off.data();
        b.ev_ts = ev_ts.data();
        b.ev_feat_off = ev_feat_off.data();
        b.ev_feats = ev_feats.data();
        b.exp_off = exp_off.data();
        b.exp_scenario = exp_scenario.data();
        b.exp_ts = exp_ts.data();
        b.exp_feat_off = exp_feat_off.data();
        b.exp_blk = exp_blk.data();
        b.exp_feats = exp_feats.data();
        return b;
    }
};

class GpuModel {
  public:
    // Mirrors Model<Real>::build: config + schema set, then every ParamStore
    // entry uploaded by its registered name (model.hpp:371-463).
    template <typename Real>
    explicit GpuModel(const Model<Real>& model, int device = 0, int32_t precision = MTFM_PRECISION_BF16)
        : schemas_(model.schemas) {
        init(model.cfg, model.params, device, precision, -1);
    }
    // A scenario deployment: ScenarioSubgraph<Real> from extract_subgraph(model, s)
    // (subgraph.hpp:12-42) — only the subgraph's ParamStore (shared weights + scenario s)
    // exists and is uploaded; every forward is scoped to s.
    template <typename Sub, typename = decltype(std::declval<const Sub&>().scenario_id)>
    explicit GpuModel(const Sub& sub, int device = 0, int32_t precision = MTFM_PRECISION_BF16)
        : schemas_(sub.schemas), subgraph_(sub.scenario_id) {
        init(sub.cfg, sub.params, device, precision, sub.scenario_id);
    }

  private:
    template <typename Store>
    void init(const ModelConfig& cfg, const Store& params, int device, int32_t precision, int subgraph) {
        const HTAConfig& h = cfg.hta;
        mtfm_model_desc md{h.d_model, h.blocks, h.target_layers, h.full_layers, h.heads, h.kv_heads,
                           static_cast<int32_t>(h.norm), h.eps, cfg.d_emb, cfg.experts, cfg.d_expert};
        std::vector<int32_t> hid, hns, hv, rid, rns, rv, sid, nu, nc, ni, sv, nt;
        std::vector<const char*> tasks;
        for (const auto& s : schemas_.hist) {
            hid.push_back(s.seq_id);
            hns.push_back(static_cast<int32_t>(s.feature_vocabs.size()));
            hv.insert(hv.end(), s.feature_vocabs.begin(), s.feature_vocabs.end());
        }
        for (const auto& s : schemas_.rt) {
            rid.push_back(s.seq_id);
            rns.push_back(static_cast<int32_t>(s.feature_vocabs.size()));
            rv.insert(rv.end(), s.feature_vocabs.begin(), s.feature_vocabs.end());
        }
        for (const auto& s : schemas_.scenarios) {
            sid.push_back(s.scenario_id);
            nu.push_back(static_cast<int32_t>(s.user_feature_vocabs.size()));
            nc.push_back(static_cast<int32_t>(s.cross_feature_vocabs.size()));
            ni.push_back(static_cast<int32_t>(s.item_feature_vocabs.size()));
            sv.insert(sv.end(), s.user_feature_vocabs.begin(), s.user_feature_vocabs.end());
            sv.insert(sv.end(), s.cross_feature_vocabs.begin(), s.cross_feature_vocabs.end());
            sv.insert(sv.end(), s.item_feature_vocabs.begin(), s.item_feature_vocabs.end());
            nt.push_back(static_cast<int32_t>(s.tasks.size()));
            for (const auto& t : s.tasks) tasks.push_back(t.c_str());
        }
        mtfm_schema_desc sd{static_cast<int32_t>(hid.size()), hid.data(), hns.data(), hv.data(),
                            static_cast<int32_t>(rid.size()), rid.data(), rns.data(), rv.data(),
                            static_cast<int32_t>(sid.size()), sid.data(), nu.data(), nc.data(), ni.data(),
                            sv.data(), nt.data(), tasks.data()};
        check(mtfm_cuda_create(device, &md, &sd, precision, &h_));
        if (subgraph >= 0) check(mtfm_cuda_restrict_to_scenario(h_, subgraph));
        std::vector<float> buf;
        for (const auto& e : params) {
            buf.assign(e.value.size(), 0.f);
            for (size_t i = 0; i < buf.size(); ++i) buf[i] = static_cast<float>(e.value[i]);
            check(mtfm_cuda_set_param(h_, e.name.c_str(), buf.data(), static_cast<int64_t>(e.value.rows()),
                                      static_cast<int64_t>(e.value.cols())));
        }
    }
  public:
    ~GpuModel() {
        if (h_) mtfm_cuda_destroy(h_);
    }
    GpuModel(const GpuModel&) = delete;
    GpuModel& operator=(const GpuModel&) = delete;

    // Concatenated Model::forward_scoped(store, s, only_scenario) records of
    // every sample, in order (model.hpp:265-312).
    std::vector<PredictionRecord> forward_samples(std::span<const UserSample> samples, int only_scenario = -1,
                                                  bool attach_labels = true) const {
        PackedBatch pb;
        for (const auto& s : samples) pb.add(s);
        const mtfm_packed_batch b = pb.view();
        const int64_t n = mtfm_cuda_count_records(h_, &b);
        std::vector<int64_t> uid(static_cast<size_t>(n));
        std::vector<int32_t> scen(static_cast<size_t>(n)), exp(static_cast<size_t>(n)), task(static_cast<size_t>(n));
        std::vector<double> prob(static_cast<size_t>(n));
        mtfm_records out{n, 0, uid.data(), scen.data(), exp.data(), task.data(), nullptr, prob.data()};
        check(mtfm_cuda_forward(h_, &b, only_scenario, &out));
        std::vector<PredictionRecord> recs;
        recs.reserve(static_cast<size_t>(out.n_records));
        size_t si = 0, left = 0;
        for (int64_t i = 0; i < out.n_records; ++i) {
            // records are user-major in batch order: find the sample owning record i
            while (left == 0 && si < samples.size()) {
                for (const auto& e : samples[si].exposures)
                    if (only_scenario < 0 || e.scenario_id == only_scenario)
                        left += schemas_.scenario(e.scenario_id).tasks.size();
                if (left == 0) ++si;
            }
            PredictionRecord r;
            r.user_id = uid[static_cast<size_t>(i)];
            r.scenario_id = scen[static_cast<size_t>(i)];
            r.exposure_index = exp[static_cast<size_t>(i)];
            r.task = schemas_.scenario(r.scenario_id).tasks[static_cast<size_t>(task[static_cast<size_t>(i)])];
            r.probability = prob[static_cast<size_t>(i)];
            if (attach_labels) {
                const auto& labels = samples[si].exposures[static_cast<size_t>(r.exposure_index)].labels;
                auto it = labels.find(r.task);
                r.label = it == labels.end() ? -1 : it->second;
            }
            recs.push_back(std::move(r));
            if (--left == 0) ++si;
        }
        return recs;
    }

    std::vector<PredictionRecord> forward_sample(const UserSample& s) const {
        return forward_samples(std::span<const UserSample>(&s, 1));
    }

    // subgraph.hpp:47-62: all candidates of the request scored in one sequence,
    // bound to the request's scenario only, no labels.
    std::vector<PredictionRecord> infer_request(const InferenceRequest& r) const {
        const UserSample view = sample_view_of_request(r);
        return forward_samples(std::span<const UserSample>(&view, 1), r.scenario_id, false);
    }

    // Many requests in ONE forward (each request one sample of the batch); per request
    // the records equal infer_request(r): T tokens never see other users or each other.
    std::vector<std::vector<PredictionRecord>> infer_requests(std::span<const InferenceRequest> rs) const {
        std::vector<UserSample> views;
        views.reserve(rs.size());
        for (const auto& r : rs) {
            if (subgraph_ >= 0 && r.scenario_id != subgraph_)
                throw integrity_error("request scenario " + std::to_string(r.scenario_id) +
                                      " does not match subgraph scenario " + std::to_string(subgraph_));
            views.push_back(sample_view_of_request(r));
        }
        auto flat = forward_samples(std::span<const UserSample>(views.data(), views.size()), subgraph_, false);
        std::vector<std::vector<PredictionRecord>> out(rs.size());
        size_t k = 0;
        for (size_t i = 0; i < rs.size(); ++i) {
            const size_t n = rs[i].candidates.size() * schemas_.scenario(rs[i].scenario_id).tasks.size();
            out[i].assign(flat.begin() + static_cast<long>(k), flat.begin() + static_cast<long>(k + n));
            k += n;
        }
        return out;
    }

    mtfm_cuda_model* handle() const { return h_; }

  private:
    SchemaSet schemas_;
    int subgraph_ = -1;
    mtfm_cuda_model* h_ = nullptr;
};

}  // namespace cuda
}  // namespace mtfm
