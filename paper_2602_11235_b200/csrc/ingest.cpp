// ingest.cpp — load_dataset (proj/src/dataset_io.cpp:110-221) straight into
// packed jagged batches: the reference's line-delimited dataset text (a header
// object with the schemas, then one UserSample object per line) parsed by
// worker threads into per-chunk packed arrays (include/mtfm_cuda.h layout) in
// page-locked memory, so each chunk goes to the GPU by an asynchronous H2D
// without re-packing per-user objects (the paper's CPU-GPU
// overlap).
//
// Semantics follow the reference exactly: every object must carry exactly its
// key set (require_keys, dataset_io.cpp:16-31: the first missing key in key
// list order, else the first unknown key in sorted order), errors are
// parse_error "line N: ..." for the first malformed line of the file, then
// validate_dataset (schema.cpp:45-139) in its order: schemas, then samples in
// file order with validate_sample's check order. Labels come out per exposure
// and task (schema task order, -1 when absent).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/mtfm_cuda.h"

namespace mtfm {
void set_last_error(const std::string& what);  // model.cu
}

namespace {

struct Fail : std::runtime_error {
    mtfm_status st;
    long line;
    Fail(mtfm_status s, const std::string& m, long l = 0) : std::runtime_error(m), st(s), line(l) {}
};

// ---------------------------------------------------------------- JSON subset
// Objects, arrays, integers, strings (the dataset's value types). Objects are
// read into (key, value span) lists so key sets can be checked like
// require_keys before any value is converted.
struct Cur {
    const char* p;
    const char* e;
};

void ws(Cur& c) {
    while (c.p < c.e && (*c.p == ' ' || *c.p == '\t' || *c.p == '\r' || *c.p == '\n')) ++c.p;
}

[[noreturn]] void bad(const char* what) { throw Fail(MTFM_PARSE_ERROR, what); }

void skip_string(Cur& c) {
    if (c.p >= c.e || *c.p != '"') bad("syntax error: expected string");
    ++c.p;
    while (c.p < c.e && *c.p != '"') {
        if (*c.p == '\\') ++c.p;
        ++c.p;
    }
    if (c.p >= c.e) bad("syntax error: unterminated string");
    ++c.p;
}

std::string read_string(Cur& c) {
    ws(c);
    if (c.p >= c.e || *c.p != '"') bad("type must be string");
    ++c.p;
    std::string out;
    while (c.p < c.e && *c.p != '"') {
        if (*c.p == '\\') {
            ++c.p;
            if (c.p >= c.e) break;
            const char q = *c.p;
            out.push_back(q == 'n' ? '\n' : q == 't' ? '\t' : q == 'r' ? '\r' : q == 'b' ? '\b' : q == 'f' ? '\f' : q);
        } else {
            out.push_back(*c.p);
        }
        ++c.p;
    }
    if (c.p >= c.e) bad("syntax error: unterminated string");
    ++c.p;
    return out;
}

void skip_value(Cur& c);

void skip_container(Cur& c, char open, char close) {
    ++c.p;
    ws(c);
    if (c.p < c.e && *c.p == close) {
        ++c.p;
        return;
    }
    for (;;) {
        ws(c);
        if (open == '{') {
            skip_string(c);
            ws(c);
            if (c.p >= c.e || *c.p != ':') bad("syntax error: expected ':'");
            ++c.p;
        }
        skip_value(c);
        ws(c);
        if (c.p < c.e && *c.p == ',') {
            ++c.p;
            continue;
        }
        if (c.p < c.e && *c.p == close) {
            ++c.p;
            return;
        }
        bad("syntax error: expected ',' or closing bracket");
    }
}

void skip_value(Cur& c) {
    ws(c);
    if (c.p >= c.e) bad("syntax error: unexpected end of input");
    const char ch = *c.p;
    if (ch == '{') return skip_container(c, '{', '}');
    if (ch == '[') return skip_container(c, '[', ']');
    if (ch == '"') return skip_string(c);
    const char* s = c.p;
    while (c.p < c.e && (std::isalnum(static_cast<unsigned char>(*c.p)) || *c.p == '-' || *c.p == '+' || *c.p == '.'))
        ++c.p;
    if (c.p == s) bad("syntax error: unexpected character");
}

struct Obj {
    std::vector<std::pair<std::string, Cur>> kv;  // last value wins for duplicate keys (nlohmann)
    const Cur* get(const char* k) const {
        for (size_t i = kv.size(); i-- > 0;)
            if (kv[i].first == k) return &kv[i].second;
        return nullptr;
    }
};

Obj read_object(Cur& c) {
    ws(c);
    if (c.p >= c.e || *c.p != '{') bad("expected object");
    Obj o;
    ++c.p;
    ws(c);
    if (c.p < c.e && *c.p == '}') {
        ++c.p;
        return o;
    }
    for (;;) {
        std::string k = read_string(c);
        ws(c);
        if (c.p >= c.e || *c.p != ':') bad("syntax error: expected ':'");
        ++c.p;
        ws(c);
        Cur v{c.p, c.e};
        skip_value(c);
        v.e = c.p;
        o.kv.emplace_back(std::move(k), v);
        ws(c);
        if (c.p < c.e && *c.p == ',') {
            ++c.p;
            ws(c);
            continue;
        }
        if (c.p < c.e && *c.p == '}') {
            ++c.p;
            return o;
        }
        bad("syntax error: expected ',' or '}'");
    }
}

// require_keys (dataset_io.cpp:16-31)
void require_keys(const Obj& o, std::initializer_list<const char*> keys) {
    for (const char* k : keys)
        if (!o.get(k)) throw Fail(MTFM_PARSE_ERROR, std::string("missing key '") + k + "'");
    std::set<std::string> uniq;
    for (const auto& kv : o.kv) uniq.insert(kv.first);
    if (uniq.size() != keys.size())
        for (const auto& k : uniq) {  // std::map order, as nlohmann iterates
            bool known = false;
            for (const char* q : keys) known = known || k == q;
            if (!known) throw Fail(MTFM_PARSE_ERROR, "unknown key '" + k + "'");
        }
}

int64_t read_int(Cur c) {
    ws(c);
    if (c.p >= c.e) bad("type must be number");
    if (*c.p == '"' || *c.p == '[' || *c.p == '{' || *c.p == 't' || *c.p == 'f' || *c.p == 'n')
        bad("type must be number");
    bool neg = false;
    if (*c.p == '-') {
        neg = true;
        ++c.p;
    }
    int64_t v = 0;
    const char* s = c.p;
    while (c.p < c.e && *c.p >= '0' && *c.p <= '9') v = v * 10 + (*c.p++ - '0');
    if (c.p == s) bad("type must be number");
    // number_float -> integer conversion truncates toward zero (nlohmann get<int>)
    if (c.p < c.e && (*c.p == '.' || *c.p == 'e' || *c.p == 'E')) {
        const double d = std::strtod(s - (neg ? 1 : 0), nullptr);
        return static_cast<int64_t>(d);
    }
    return neg ? -v : v;
}

template <typename F>
void for_array(Cur c, F&& f) {
    ws(c);
    if (c.p >= c.e || *c.p != '[') bad("type must be array");
    ++c.p;
    ws(c);
    if (c.p < c.e && *c.p == ']') return;
    for (;;) {
        ws(c);
        Cur v{c.p, c.e};
        skip_value(c);
        v.e = c.p;
        f(v);
        ws(c);
        if (c.p < c.e && *c.p == ',') {
            ++c.p;
            continue;
        }
        if (c.p < c.e && *c.p == ']') return;
        bad("syntax error: expected ',' or ']'");
    }
}

std::vector<int> read_ints(const Cur& c) {
    std::vector<int> out;
    for_array(c, [&](const Cur& v) { out.push_back(static_cast<int>(read_int(v))); });
    return out;
}

// ---------------------------------------------------------------- schemas
struct SeqSchema {
    int id;
    std::vector<int> vocabs;
};
struct ScenSchema {
    int id;
    std::vector<int> u, c, i;
    std::vector<std::string> tasks;
};

struct Schemas {
    std::vector<SeqSchema> hist, rt;
    std::vector<ScenSchema> scen;
    const SeqSchema* hist_of(int id) const {
        for (const auto& s : hist)
            if (s.id == id) return &s;
        return nullptr;
    }
    const SeqSchema* rt_of(int id) const {
        for (const auto& s : rt)
            if (s.id == id) return &s;
        return nullptr;
    }
    const ScenSchema* scen_of(int id) const {
        for (const auto& s : scen)
            if (s.id == id) return &s;
        return nullptr;
    }
};

// ---------------------------------------------------------------- chunks
template <typename T>
struct HostArr {  // page-locked when a CUDA device is present, else malloc
    T* p = nullptr;
    size_t n = 0;
    bool pinned = false;
    HostArr() = default;
    HostArr(const HostArr&) = delete;
    HostArr& operator=(const HostArr&) = delete;
    ~HostArr() { release(); }
    void release() {
        if (p) {
            if (pinned) cudaFreeHost(p);
            else std::free(p);
        }
        p = nullptr;
        n = 0;
    }
    void assign(const std::vector<T>& v) {
        release();
        n = v.size();
        const size_t bytes = std::max<size_t>(n * sizeof(T), 16);
        if (cudaMallocHost(reinterpret_cast<void**>(&p), bytes) == cudaSuccess) {
            pinned = true;
        } else {
            cudaGetLastError();
            p = static_cast<T*>(std::malloc(bytes));
            pinned = false;
            if (!p) throw Fail(MTFM_CONTRACT_ERROR, "out of host memory");
        }
        if (n) std::memcpy(p, v.data(), n * sizeof(T));
    }
};

struct Pack {  // vectors while parsing
    std::vector<int64_t> user_id, ev_ts, exp_ts;
    std::vector<int32_t> seq_off{0}, seq_schema, ev_off{0}, ev_feat_off{0}, ev_feats, exp_off{0}, exp_scenario,
        exp_feat_off{0}, exp_blk, exp_feats, labels;
    std::vector<uint8_t> seq_kind;
};

struct Chunk {
    long first_line = 0;
    int64_t n_users = 0;
    HostArr<int64_t> user_id, ev_ts, exp_ts;
    HostArr<int32_t> seq_off, seq_schema, ev_off, ev_feat_off, ev_feats, exp_off, exp_scenario, exp_feat_off, exp_blk,
        exp_feats, labels;
    HostArr<uint8_t> seq_kind;
};

struct SampleErr {  // first validation failure of a chunk: (sample index, status, message)
    int64_t sample = -1;
    mtfm_status st = MTFM_OK;
    std::string msg;
};

// One user line -> appended to the pack; validate_sample (schema.cpp:104-139) in its order.
void parse_sample(const Schemas& sch, int max_tasks, Cur line, Pack& pk, SampleErr& verr, int64_t sample_idx) {
    Obj o = read_object(line);
    require_keys(o, {"user_id", "hist", "rt", "exposures"});
    const int64_t uid = read_int(*o.get("user_id"));
    struct Ev {
        std::vector<int> f;
        int64_t t;
    };
    struct Rec {
        int seq;
        std::vector<Ev> ev;
    };
    auto seqs = [&](const Cur& c) {
        std::vector<Rec> out;
        Cur a = c;
        ws(a);
        if (a.p >= a.e || *a.p != '[') throw Fail(MTFM_PARSE_ERROR, "sequence list must be an array");
        for_array(c, [&](const Cur& rv) {
            Cur rc = rv;
            Obj r = read_object(rc);
            require_keys(r, {"seq", "events"});
            Rec rec;
            rec.seq = static_cast<int>(read_int(*r.get("seq")));
            for_array(*r.get("events"), [&](const Cur& evc) {
                Cur ec = evc;
                Obj ev = read_object(ec);
                require_keys(ev, {"f", "t"});
                rec.ev.push_back({read_ints(*ev.get("f")), read_int(*ev.get("t"))});
            });
            out.push_back(std::move(rec));
        });
        return out;
    };
    std::vector<Rec> hist = seqs(*o.get("hist")), rt = seqs(*o.get("rt"));
    struct Ex {
        int s;
        std::vector<int> u, c, i;
        int64_t t;
        std::vector<std::pair<std::string, int>> y;
    };
    std::vector<Ex> exps;
    for_array(*o.get("exposures"), [&](const Cur& xc) {
        Cur cc = xc;
        Obj e = read_object(cc);
        require_keys(e, {"s", "u", "c", "i", "t", "y"});
        Ex x;
        x.s = static_cast<int>(read_int(*e.get("s")));
        x.u = read_ints(*e.get("u"));
        x.c = read_ints(*e.get("c"));
        x.i = read_ints(*e.get("i"));
        x.t = read_int(*e.get("t"));
        Cur yc = *e.get("y");
        Obj y = read_object(yc);
        for (const auto& kv : y.kv) {
            int v = static_cast<int>(read_int(kv.second));
            bool dup = false;
            for (auto& p : x.y)
                if (p.first == kv.first) {
                    p.second = v;
                    dup = true;
                }
            if (!dup) x.y.emplace_back(kv.first, v);
        }
        exps.push_back(std::move(x));
    });
    // ---- validate_sample (first failure of the chunk is kept; parsing continues)
    if (verr.sample < 0) {
        auto fail = [&](mtfm_status st, const std::string& m) {
            verr.sample = sample_idx;
            verr.st = st;
            verr.msg = m;
        };
        const std::string who = "user " + std::to_string(uid);
        auto check = [&]() -> bool {
            if (exps.empty()) return fail(MTFM_INTEGRITY_ERROR, who + ": no exposures"), false;
            int64_t min_ts = exps.front().t;
            for (const auto& e : exps) min_ts = std::min(min_ts, e.t);
            auto events = [&](const SeqSchema& s, const Rec& rec) -> bool {
                int64_t prev = -1;
                for (const auto& ev : rec.ev) {
                    if (ev.t < 0) return fail(MTFM_INTEGRITY_ERROR, who + ": negative timestamp"), false;
                    if (ev.t < prev)
                        return fail(MTFM_INTEGRITY_ERROR,
                                    who + ": events not sorted by timestamp in sequence " + std::to_string(rec.seq)),
                               false;
                    prev = ev.t;
                    if (ev.f.size() != s.vocabs.size())
                        return fail(MTFM_INTEGRITY_ERROR,
                                    who + ": event feature count mismatch in sequence " + std::to_string(rec.seq)),
                               false;
                    for (size_t k = 0; k < ev.f.size(); ++k)
                        if (ev.f[k] < 0 || ev.f[k] >= s.vocabs[k])
                            return fail(MTFM_LOOKUP_ERROR, who + ": feature id " + std::to_string(ev.f[k]) +
                                                               " out of vocab range"),
                                   false;
                }
                return true;
            };
            for (const auto& rec : hist) {
                const SeqSchema* s = sch.hist_of(rec.seq);
                if (!s)
                    return fail(MTFM_INTEGRITY_ERROR, "unknown historical sequence schema " + std::to_string(rec.seq)),
                           false;
                if (!events(*s, rec)) return false;
                for (const auto& ev : rec.ev)
                    if (ev.t >= min_ts)
                        return fail(MTFM_INTEGRITY_ERROR, who + ": historical event at or after first exposure"), false;
            }
            for (const auto& rec : rt) {
                const SeqSchema* s = sch.rt_of(rec.seq);
                if (!s)
                    return fail(MTFM_INTEGRITY_ERROR, "unknown realtime sequence schema " + std::to_string(rec.seq)),
                           false;
                if (!events(*s, rec)) return false;
            }
            for (const auto& e : exps) {
                const ScenSchema* sc = sch.scen_of(e.s);
                if (!sc) return fail(MTFM_INTEGRITY_ERROR, "unknown scenario id " + std::to_string(e.s)), false;
                auto block = [&](const std::vector<int>& ids, const std::vector<int>& voc, const char* which) -> bool {
                    if (ids.size() != voc.size())
                        return fail(MTFM_INTEGRITY_ERROR, who + ": " + which + " feature count mismatch"), false;
                    for (size_t k = 0; k < ids.size(); ++k)
                        if (ids[k] < 0 || ids[k] >= voc[k])
                            return fail(MTFM_LOOKUP_ERROR, who + ": " + which + " feature id " + std::to_string(ids[k]) +
                                                               " out of vocab range"),
                                   false;
                    return true;
                };
                if (!block(e.u, sc->u, "user") || !block(e.c, sc->c, "cross") || !block(e.i, sc->i, "item"))
                    return false;
                if (e.t < 0) return fail(MTFM_INTEGRITY_ERROR, who + ": negative exposure timestamp"), false;
                auto label = [&](const std::string& t) -> const int* {
                    for (const auto& p : e.y)
                        if (p.first == t) return &p.second;
                    return nullptr;
                };
                for (const auto& t : sc->tasks) {
                    const int* v = label(t);
                    if (!v) return fail(MTFM_INTEGRITY_ERROR, who + ": missing label for " + t), false;
                    if (*v != 0 && *v != 1) return fail(MTFM_INTEGRITY_ERROR, who + ": non-binary label for " + t), false;
                }
                const bool has_ctr = std::find(sc->tasks.begin(), sc->tasks.end(), "ctr") != sc->tasks.end();
                const bool has_ctcvr = std::find(sc->tasks.begin(), sc->tasks.end(), "ctcvr") != sc->tasks.end();
                if (has_ctr && has_ctcvr && *label("ctcvr") == 1 && *label("ctr") == 0)
                    return fail(MTFM_INTEGRITY_ERROR, who + ": funnel violation, ctcvr=1 with ctr=0"), false;
            }
            return true;
        };
        check();
    }
    // ---- pack (schema.py pack_samples layout)
    pk.user_id.push_back(uid);
    auto eat = [&](const std::vector<Rec>& v, uint8_t kind) {
        for (const auto& rec : v) {
            pk.seq_kind.push_back(kind);
            pk.seq_schema.push_back(rec.seq);
            for (const auto& ev : rec.ev) {
                pk.ev_ts.push_back(ev.t);
                pk.ev_feats.insert(pk.ev_feats.end(), ev.f.begin(), ev.f.end());
                pk.ev_feat_off.push_back(static_cast<int32_t>(pk.ev_feats.size()));
            }
            pk.ev_off.push_back(static_cast<int32_t>(pk.ev_ts.size()));
        }
    };
    eat(hist, 0);
    eat(rt, 1);
    pk.seq_off.push_back(static_cast<int32_t>(pk.seq_kind.size()));
    for (const auto& e : exps) {
        pk.exp_scenario.push_back(e.s);
        pk.exp_ts.push_back(e.t);
        pk.exp_blk.push_back(static_cast<int32_t>(e.u.size()));
        pk.exp_blk.push_back(static_cast<int32_t>(e.c.size()));
        pk.exp_blk.push_back(static_cast<int32_t>(e.i.size()));
        pk.exp_feats.insert(pk.exp_feats.end(), e.u.begin(), e.u.end());
        pk.exp_feats.insert(pk.exp_feats.end(), e.c.begin(), e.c.end());
        pk.exp_feats.insert(pk.exp_feats.end(), e.i.begin(), e.i.end());
        pk.exp_feat_off.push_back(static_cast<int32_t>(pk.exp_feats.size()));
        const ScenSchema* sc = sch.scen_of(e.s);
        for (int t = 0; t < max_tasks; ++t) {
            int v = -1;
            if (sc && t < static_cast<int>(sc->tasks.size()))
                for (const auto& p : e.y)
                    if (p.first == sc->tasks[static_cast<size_t>(t)]) v = p.second;
            pk.labels.push_back(v);
        }
    }
    pk.exp_off.push_back(static_cast<int32_t>(pk.exp_scenario.size()));
}

}  // namespace

struct mtfm_dataset {
    int format_version = 1;
    Schemas sch;
    int max_tasks = 0;
    int64_t n_users = 0;
    std::vector<std::unique_ptr<Chunk>> chunks;
    // schema desc storage (mtfm_dataset_schema_desc)
    std::vector<int32_t> hid, hns, hv, rid, rns, rv, sid, nu, nc, ni, sv, nt;
    std::vector<const char*> tasks;
};

extern "C" {

mtfm_status mtfm_dataset_load(const char* path, int32_t n_threads, int32_t chunk_users, mtfm_dataset** out) {
    try {
        if (!path || !out) throw Fail(MTFM_CONTRACT_ERROR, "null argument");
        if (chunk_users < 1) throw Fail(MTFM_CONTRACT_ERROR, "chunk_users must be >= 1");
        std::ifstream in(path, std::ios::binary);
        if (!in) throw Fail(MTFM_CONFIG_ERROR, std::string("cannot open dataset: ") + path);
        std::string bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
        // line index
        std::vector<std::pair<size_t, size_t>> lines;
        for (size_t p = 0; p < bytes.size();) {
            size_t q = bytes.find('\n', p);
            if (q == std::string::npos) q = bytes.size();
            lines.emplace_back(p, q);
            p = q + 1;
        }
        if (lines.empty()) throw Fail(MTFM_PARSE_ERROR, "line 1: empty input, missing header");
        auto D = std::make_unique<mtfm_dataset>();
        // header (dataset_io.cpp:150-168)
        try {
            Cur c{bytes.data() + lines[0].first, bytes.data() + lines[0].second};
            Obj h = read_object(c);
            require_keys(h, {"format", "version", "hist_seq_schemas", "rt_seq_schemas", "scenarios"});
            Cur fc = *h.get("format");
            if (read_string(fc) != "mtfm-dataset") throw Fail(MTFM_PARSE_ERROR, "not a mtfm dataset file");
            D->format_version = static_cast<int>(read_int(*h.get("version")));
            auto seq = [&](const Cur& arr, std::vector<SeqSchema>& dst) {
                for_array(arr, [&](const Cur& v) {
                    Cur vc = v;
                    Obj o = read_object(vc);
                    require_keys(o, {"seq_id", "vocabs"});
                    dst.push_back({static_cast<int>(read_int(*o.get("seq_id"))), read_ints(*o.get("vocabs"))});
                });
            };
            seq(*h.get("hist_seq_schemas"), D->sch.hist);
            seq(*h.get("rt_seq_schemas"), D->sch.rt);
            for_array(*h.get("scenarios"), [&](const Cur& v) {
                Cur vc = v;
                Obj o = read_object(vc);
                require_keys(o, {"scenario_id", "user_vocabs", "cross_vocabs", "item_vocabs", "tasks"});
                ScenSchema s;
                s.id = static_cast<int>(read_int(*o.get("scenario_id")));
                s.u = read_ints(*o.get("user_vocabs"));
                s.c = read_ints(*o.get("cross_vocabs"));
                s.i = read_ints(*o.get("item_vocabs"));
                for_array(*o.get("tasks"), [&](const Cur& t) {
                    Cur tc = t;
                    s.tasks.push_back(read_string(tc));
                });
                D->sch.scen.push_back(std::move(s));
            });
        } catch (const Fail& f) {
            if (f.st != MTFM_PARSE_ERROR) throw;
            std::string m = f.what();
            if (m.rfind("missing key", 0) != 0 && m.rfind("unknown key", 0) != 0 && m != "not a mtfm dataset file" &&
                m != "expected object")
                m = "malformed header: " + m;
            throw Fail(MTFM_PARSE_ERROR, "line 1: " + m, 1);
        }
        for (const auto& s : D->sch.scen) D->max_tasks = std::max(D->max_tasks, static_cast<int>(s.tasks.size()));
        // sample lines (empty lines skipped, line numbers kept), chunked by users
        std::vector<long> sample_lines;
        for (size_t k = 1; k < lines.size(); ++k)
            if (lines[k].second > lines[k].first) sample_lines.push_back(static_cast<long>(k));
        const int64_t U = static_cast<int64_t>(sample_lines.size());
        const int64_t n_chunks = (U + chunk_users - 1) / chunk_users;
        D->n_users = U;
        D->chunks.resize(static_cast<size_t>(n_chunks));
        std::vector<long> perr_line(static_cast<size_t>(n_chunks), 0);
        std::vector<std::string> perr_msg(static_cast<size_t>(n_chunks));
        std::vector<SampleErr> verr(static_cast<size_t>(n_chunks));
        std::atomic<int64_t> next{0};
        auto worker = [&]() {
            for (int64_t ci; (ci = next.fetch_add(1)) < n_chunks;) {
                Pack pk;
                const int64_t u0 = ci * chunk_users, u1 = std::min(U, u0 + chunk_users);
                auto ch = std::make_unique<Chunk>();
                for (int64_t u = u0; u < u1; ++u) {
                    const long ln = sample_lines[static_cast<size_t>(u)];
                    Cur c{bytes.data() + lines[static_cast<size_t>(ln)].first, bytes.data() + lines[static_cast<size_t>(ln)].second};
                    try {
                        parse_sample(D->sch, D->max_tasks, c, pk, verr[static_cast<size_t>(ci)], u);
                    } catch (const Fail& f) {
                        std::string m = f.what();
                        if (m.rfind("missing key", 0) != 0 && m.rfind("unknown key", 0) != 0 && m != "expected object" &&
                            m != "sequence list must be an array")
                            m = "malformed record: " + m;
                        perr_line[static_cast<size_t>(ci)] = ln + 1;
                        perr_msg[static_cast<size_t>(ci)] = "line " + std::to_string(ln + 1) + ": " + m;
                        break;
                    }
                }
                if (perr_line[static_cast<size_t>(ci)]) continue;
                ch->n_users = u1 - u0;
                ch->first_line = sample_lines.empty() ? 0 : sample_lines[static_cast<size_t>(u0)] + 1;
                ch->user_id.assign(pk.user_id);
                ch->seq_off.assign(pk.seq_off);
                ch->seq_kind.assign(pk.seq_kind);
                ch->seq_schema.assign(pk.seq_schema);
                ch->ev_off.assign(pk.ev_off);
                ch->ev_ts.assign(pk.ev_ts);
                ch->ev_feat_off.assign(pk.ev_feat_off);
                ch->ev_feats.assign(pk.ev_feats);
                ch->exp_off.assign(pk.exp_off);
                ch->exp_scenario.assign(pk.exp_scenario);
                ch->exp_ts.assign(pk.exp_ts);
                ch->exp_feat_off.assign(pk.exp_feat_off);
                ch->exp_blk.assign(pk.exp_blk);
                ch->exp_feats.assign(pk.exp_feats);
                ch->labels.assign(pk.labels);
                D->chunks[static_cast<size_t>(ci)] = std::move(ch);
            }
        };
        const int nt = std::max(1, std::min<int>(n_threads > 0 ? n_threads : static_cast<int>(std::thread::hardware_concurrency()),
                                                 static_cast<int>(std::max<int64_t>(n_chunks, 1))));
        std::vector<std::thread> pool;
        for (int t = 1; t < nt; ++t) pool.emplace_back(worker);
        worker();
        for (auto& t : pool) t.join();
        // deserialize_dataset: every line parses first (the first malformed line wins) ...
        for (int64_t ci = 0; ci < n_chunks; ++ci)
            if (perr_line[static_cast<size_t>(ci)]) throw Fail(MTFM_PARSE_ERROR, perr_msg[static_cast<size_t>(ci)]);
        // ... then validate_dataset: schemas (schema.cpp:45-64), then samples in order
        {
            std::set<int> seen;
            for (const auto& s : D->sch.scen) {
                if (!seen.insert(s.id).second) throw Fail(MTFM_CONFIG_ERROR, "duplicate scenario id " + std::to_string(s.id));
                if (s.tasks.empty()) throw Fail(MTFM_CONFIG_ERROR, "scenario " + std::to_string(s.id) + ": empty task list");
                auto voc = [&](const std::vector<int>& v, const char* which) {
                    for (int n : v)
                        if (n < 2)
                            throw Fail(MTFM_CONFIG_ERROR, "scenario " + std::to_string(s.id) + ": " + which + " vocab size " +
                                                              std::to_string(n) + " < 2");
                };
                voc(s.u, "user");
                voc(s.c, "cross");
                voc(s.i, "item");
            }
            auto seqc = [](const std::vector<SeqSchema>& v, const char* kind) {
                std::set<int> ids;
                for (const auto& s : v) {
                    if (!ids.insert(s.id).second)
                        throw Fail(MTFM_CONFIG_ERROR, std::string("duplicate ") + kind + " sequence schema id");
                    for (int n : s.vocabs)
                        if (n < 2) throw Fail(MTFM_CONFIG_ERROR, std::string(kind) + " sequence vocab size < 2");
                }
            };
            seqc(D->sch.hist, "historical");
            seqc(D->sch.rt, "realtime");
        }
        for (int64_t ci = 0; ci < n_chunks; ++ci)
            if (verr[static_cast<size_t>(ci)].sample >= 0)
                throw Fail(verr[static_cast<size_t>(ci)].st, verr[static_cast<size_t>(ci)].msg);
        // schema desc arrays (mtfm_dataset_schema_desc)
        for (const auto& s : D->sch.hist) {
            D->hid.push_back(s.id);
            D->hns.push_back(static_cast<int32_t>(s.vocabs.size()));
            D->hv.insert(D->hv.end(), s.vocabs.begin(), s.vocabs.end());
        }
        for (const auto& s : D->sch.rt) {
            D->rid.push_back(s.id);
            D->rns.push_back(static_cast<int32_t>(s.vocabs.size()));
            D->rv.insert(D->rv.end(), s.vocabs.begin(), s.vocabs.end());
        }
        for (const auto& s : D->sch.scen) {
            D->sid.push_back(s.id);
            D->nu.push_back(static_cast<int32_t>(s.u.size()));
            D->nc.push_back(static_cast<int32_t>(s.c.size()));
            D->ni.push_back(static_cast<int32_t>(s.i.size()));
            D->sv.insert(D->sv.end(), s.u.begin(), s.u.end());
            D->sv.insert(D->sv.end(), s.c.begin(), s.c.end());
            D->sv.insert(D->sv.end(), s.i.begin(), s.i.end());
            D->nt.push_back(static_cast<int32_t>(s.tasks.size()));
            for (const auto& t : s.tasks) D->tasks.push_back(t.c_str());
        }
        *out = D.release();
        return MTFM_OK;
    } catch (const Fail& f) {
        mtfm::set_last_error(f.what());
        return f.st;
    } catch (const std::exception& e) {
        mtfm::set_last_error(e.what());
        return MTFM_CONTRACT_ERROR;
    }
}

mtfm_status mtfm_dataset_info(const mtfm_dataset* d, mtfm_dataset_info_t* info) {
    if (!d || !info) return MTFM_CONTRACT_ERROR;
    info->format_version = d->format_version;
    info->n_users = d->n_users;
    info->n_chunks = static_cast<int64_t>(d->chunks.size());
    info->max_tasks = d->max_tasks;
    return MTFM_OK;
}

mtfm_status mtfm_dataset_schema_desc(const mtfm_dataset* d, mtfm_schema_desc* sd) {
    if (!d || !sd) return MTFM_CONTRACT_ERROR;
    sd->n_hist = static_cast<int32_t>(d->hid.size());
    sd->hist_ids = d->hid.data();
    sd->hist_nslots = d->hns.data();
    sd->hist_vocabs = d->hv.data();
    sd->n_rt = static_cast<int32_t>(d->rid.size());
    sd->rt_ids = d->rid.data();
    sd->rt_nslots = d->rns.data();
    sd->rt_vocabs = d->rv.data();
    sd->n_scen = static_cast<int32_t>(d->sid.size());
    sd->scen_ids = d->sid.data();
    sd->scen_nu = d->nu.data();
    sd->scen_nc = d->nc.data();
    sd->scen_ni = d->ni.data();
    sd->scen_vocabs = d->sv.data();
    sd->scen_ntasks = d->nt.data();
    sd->task_names = d->tasks.data();
    return MTFM_OK;
}

mtfm_status mtfm_dataset_chunk(const mtfm_dataset* d, int64_t i, mtfm_packed_batch* b, const int32_t** labels) {
    if (!d || !b || i < 0 || i >= static_cast<int64_t>(d->chunks.size())) return MTFM_CONTRACT_ERROR;
    const Chunk& c = *d->chunks[static_cast<size_t>(i)];
    b->n_users = static_cast<int32_t>(c.n_users);
    b->n_seqs = static_cast<int32_t>(c.seq_kind.n);
    b->n_events = static_cast<int32_t>(c.ev_ts.n);
    b->n_exposures = static_cast<int32_t>(c.exp_ts.n);
    b->n_ev_feats = static_cast<int64_t>(c.ev_feats.n);
    b->n_exp_feats = static_cast<int64_t>(c.exp_feats.n);
    b->user_id = c.user_id.p;
    b->seq_off = c.seq_off.p;
    b->seq_kind = c.seq_kind.p;
    b->seq_schema = c.seq_schema.p;
    b->ev_off = c.ev_off.p;
    b->ev_ts = c.ev_ts.p;
    b->ev_feat_off = c.ev_feat_off.p;
    b->ev_feats = c.ev_feats.p;
    b->exp_off = c.exp_off.p;
    b->exp_scenario = c.exp_scenario.p;
    b->exp_ts = c.exp_ts.p;
    b->exp_feat_off = c.exp_feat_off.p;
    b->exp_blk = c.exp_blk.p;
    b->exp_feats = c.exp_feats.p;
    if (labels) *labels = c.labels.p;
    return MTFM_OK;
}

void mtfm_dataset_free(mtfm_dataset* d) { delete d; }

}  // extern "C"
