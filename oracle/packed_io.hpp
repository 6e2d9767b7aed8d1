// packed_io.hpp — reads the MTFMPB1 packed batch / MTFMPF1 parameter files
// (paper_2602_11235_b200/packed_io.py) into the reference's own types
// (mtfm::Dataset / UserSample, ModelConfig, ParamStore values).
//
// TEST / BASELINE INFRASTRUCTURE ONLY: lets the reference CPU path
// (ref_bench, ref_dump) score byte-identical inputs to the GPU path.
#pragma once

#include <cstdint>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "mtfm/model.hpp"
#include "mtfm/schema.hpp"

namespace mtfa {

struct PackedArrays {
    std::vector<int64_t> user_id, ev_ts, exp_ts;
    std::vector<int32_t> seq_off, seq_schema, ev_off, ev_feat_off, ev_feats, exp_off, exp_scenario, exp_feat_off,
        exp_blk, exp_feats;
    std::vector<uint8_t> seq_kind;
};

struct PackedFile {
    bool has_model = false;
    mtfm::ModelConfig cfg;
    mtfm::Dataset data;  // schemas + samples (labels empty)
    PackedArrays a;
};

inline std::vector<std::string> split_line(std::istream& in) {
    std::string s;
    if (!std::getline(in, s)) throw mtfm::parse_error("packed file: truncated header");
    std::istringstream is(s);
    std::vector<std::string> out;
    for (std::string w; is >> w;) out.push_back(w);
    return out;
}

template <typename T>
void read_array(std::istream& in, const std::string& code, int64_t n, std::vector<T>& dst) {
    const size_t el = code == "u1" || code == "i1" ? 1 : code == "i4" ? 4 : 8;
    if (el != sizeof(T)) throw mtfm::parse_error("packed file: dtype mismatch");
    dst.resize(static_cast<size_t>(n));
    in.read(reinterpret_cast<char*>(dst.data()), static_cast<std::streamsize>(n * el));
    if (!in) throw mtfm::parse_error("packed file: truncated array");
}

inline PackedFile load_packed(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw mtfm::parse_error("cannot open " + path);
    PackedFile pf;
    auto magic = split_line(in);
    if (magic.empty() || magic[0] != "MTFMPB1") throw mtfm::parse_error(path + ": not an MTFMPB1 file");
    auto m = split_line(in);
    if (m.size() > 1 && m[1] != "-") {
        pf.has_model = true;
        auto& h = pf.cfg.hta;
        h.d_model = std::stoi(m[1]);
        h.blocks = std::stoi(m[2]);
        h.target_layers = std::stoi(m[3]);
        h.full_layers = std::stoi(m[4]);
        h.heads = std::stoi(m[5]);
        h.kv_heads = std::stoi(m[6]);
        const int norm = std::stoi(m[7]);
        h.norm = norm == 0 ? mtfm::AttnNorm::valid_count : (norm == 1 ? mtfm::AttnNorm::seq_len : mtfm::AttnNorm::none);
        h.eps = std::stod(m[8]);
        pf.cfg.d_emb = std::stoi(m[9]);
        pf.cfg.experts = std::stoi(m[10]);
        pf.cfg.d_expert = std::stoi(m[11]);
    }
    for (int tag = 0; tag < 2; ++tag) {
        auto h = split_line(in);
        const int n = std::stoi(h.at(1));
        for (int i = 0; i < n; ++i) {
            auto v = split_line(in);
            mtfm::SequenceSchema s;
            s.seq_id = std::stoi(v.at(0));
            const int ns = std::stoi(v.at(1));
            for (int k = 0; k < ns; ++k) s.feature_vocabs.push_back(std::stoi(v.at(2 + k)));
            (tag == 0 ? pf.data.hist_seq_schemas : pf.data.rt_seq_schemas).push_back(s);
        }
    }
    {
        auto h = split_line(in);
        const int n = std::stoi(h.at(1));
        for (int i = 0; i < n; ++i) {
            auto v = split_line(in);
            mtfm::ScenarioSchema s;
            s.scenario_id = std::stoi(v.at(0));
            const int nu = std::stoi(v.at(1)), nc = std::stoi(v.at(2)), ni = std::stoi(v.at(3));
            size_t p = 4;
            for (int k = 0; k < nu; ++k) s.user_feature_vocabs.push_back(std::stoi(v.at(p++)));
            for (int k = 0; k < nc; ++k) s.cross_feature_vocabs.push_back(std::stoi(v.at(p++)));
            for (int k = 0; k < ni; ++k) s.item_feature_vocabs.push_back(std::stoi(v.at(p++)));
            const int nt = std::stoi(v.at(p++));
            for (int k = 0; k < nt; ++k) s.tasks.push_back(v.at(p++));
            pf.data.scenarios.push_back(s);
        }
    }
    auto ah = split_line(in);
    const int n_arr = std::stoi(ah.at(1));
    auto& a = pf.a;
    for (int i = 0; i < n_arr; ++i) {
        auto h = split_line(in);
        const std::string key = h.at(0), code = h.at(1);
        const int64_t n = std::stoll(h.at(2));
        if (key == "user_id") read_array(in, code, n, a.user_id);
        else if (key == "seq_off") read_array(in, code, n, a.seq_off);
        else if (key == "seq_kind") read_array(in, code, n, a.seq_kind);
        else if (key == "seq_schema") read_array(in, code, n, a.seq_schema);
        else if (key == "ev_off") read_array(in, code, n, a.ev_off);
        else if (key == "ev_ts") read_array(in, code, n, a.ev_ts);
        else if (key == "ev_feat_off") read_array(in, code, n, a.ev_feat_off);
        else if (key == "ev_feats") read_array(in, code, n, a.ev_feats);
        else if (key == "exp_off") read_array(in, code, n, a.exp_off);
        else if (key == "exp_scenario") read_array(in, code, n, a.exp_scenario);
        else if (key == "exp_ts") read_array(in, code, n, a.exp_ts);
        else if (key == "exp_feat_off") read_array(in, code, n, a.exp_feat_off);
        else if (key == "exp_blk") read_array(in, code, n, a.exp_blk);
        else if (key == "exp_feats") read_array(in, code, n, a.exp_feats);
        else throw mtfm::parse_error("packed file: unknown array " + key);
    }
    // packed CSR -> UserSample (the inverse of schema.py pack_samples)
    const size_t U = a.user_id.size();
    for (size_t u = 0; u < U; ++u) {
        mtfm::UserSample s;
        s.user_id = a.user_id[u];
        for (int q = a.seq_off[u]; q < a.seq_off[u + 1]; ++q) {
            mtfm::SequenceRecord rec;
            rec.seq_schema_id = a.seq_schema[q];
            for (int e = a.ev_off[q]; e < a.ev_off[q + 1]; ++e) {
                mtfm::BehaviorEvent ev;
                ev.timestamp = a.ev_ts[e];
                ev.item_features.assign(a.ev_feats.begin() + a.ev_feat_off[e], a.ev_feats.begin() + a.ev_feat_off[e + 1]);
                rec.events.push_back(std::move(ev));
            }
            (a.seq_kind[q] ? s.realtime_sequences : s.historical_sequences).push_back(std::move(rec));
        }
        for (int x = a.exp_off[u]; x < a.exp_off[u + 1]; ++x) {
            mtfm::Exposure e;
            e.scenario_id = a.exp_scenario[x];
            e.timestamp = a.exp_ts[x];
            const int* f = a.exp_feats.data() + a.exp_feat_off[x];
            const int nu = a.exp_blk[3 * x], nc = a.exp_blk[3 * x + 1], ni = a.exp_blk[3 * x + 2];
            e.user_features.assign(f, f + nu);
            e.cross_features.assign(f + nu, f + nu + nc);
            e.item_features.assign(f + nu + nc, f + nu + nc + ni);
            s.exposures.push_back(std::move(e));
        }
        pf.data.samples.push_back(std::move(s));
    }
    return pf;
}

// MTFMPF1: overwrite the values of a ParamStore by name (shapes must match).
template <typename Real>
void load_params_into(const std::string& path, mtfm::ParamStore<Real>& store) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw mtfm::parse_error("cannot open " + path);
    auto magic = split_line(in);
    if (magic.empty() || magic[0] != "MTFMPF1") throw mtfm::parse_error(path + ": not an MTFMPF1 file");
    const int n = std::stoi(split_line(in).at(0));
    std::vector<float> buf;
    for (int i = 0; i < n; ++i) {
        auto h = split_line(in);
        const std::string name = h.at(0);
        const size_t r = std::stoul(h.at(1)), c = std::stoul(h.at(2));
        buf.resize(r * c);
        in.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(r * c * 4));
        if (!in) throw mtfm::parse_error("params file: truncated");
        auto& t = store.at(name).value;
        if (t.rows() != r || t.cols() != c) throw mtfm::dimension_error("params file: shape mismatch for " + name);
        for (size_t k = 0; k < r * c; ++k) t.data()[k] = static_cast<Real>(buf[k]);
    }
}

}  // namespace mtfa
