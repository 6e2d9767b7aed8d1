// jitter.hpp — TEST INFRASTRUCTURE ONLY (ref_dump, ref_integration).
#pragma once

#include <string>

#include "mtfm/params.hpp"
#include "mtfm/rng.hpp"

namespace mtfm {

inline bool ends_with(const std::string& s, const std::string& t) {
    return s.size() >= t.size() && s.compare(s.size() - t.size(), t.size(), t) == 0;
}

// Moves a Model::build parameter store away from its default initialisation
// (zero biases, unit GLN gains, zero GLN biases: model.hpp:387,440-445) so the
// goldens exercise every bias, the group-indexed GLN affine lookups and O(1)
// logits. Deterministic in registration order with the reference's own Rng
// (rng.hpp:57 uniform); restated by mtfm_oracle.jitter_params:
//   .../gain            v = 1 + U(-0.2, 0.2)
//   .../gln*/.../bias   v = U(-0.1, 0.1)
//   *_b, mlp_b1, mlp_b2 v = v + U(-0.1, 0.1)
//   .../tower_w         v = v * tower_scale
// every value computed in double, then rounded to float.
inline void jitter_params(ParamStore<float>& ps, uint64_t seed, double tower_scale) {
    Rng rng(seed);
    for (size_t k = 0; k < ps.size(); ++k) {
        auto& e = ps.at(k);
        const std::string& n = e.name;
        float* v = e.value.data();
        const size_t cnt = e.value.size();
        if (ends_with(n, "/gain")) {
            for (size_t i = 0; i < cnt; ++i) v[i] = static_cast<float>(1.0 + rng.uniform(-0.2, 0.2));
        } else if (n.find("/gln") != std::string::npos && ends_with(n, "/bias")) {
            for (size_t i = 0; i < cnt; ++i) v[i] = static_cast<float>(rng.uniform(-0.1, 0.1));
        } else if (ends_with(n, "_b") || ends_with(n, "/mlp_b1") || ends_with(n, "/mlp_b2")) {
            for (size_t i = 0; i < cnt; ++i) v[i] = static_cast<float>(static_cast<double>(v[i]) + rng.uniform(-0.1, 0.1));
        } else if (ends_with(n, "/tower_w")) {
            for (size_t i = 0; i < cnt; ++i) v[i] = static_cast<float>(static_cast<double>(v[i]) * tower_scale);
        }
    }
}


}  // namespace mtfm
