// mtfa.hpp — tiny named-array archive writer used by the oracle dump tools.
//
// TEST INFRASTRUCTURE ONLY (oracle/): never linked into the product library.
//
// Layout: "MTFA1\n" then per entry
//   u32 name_len, name bytes, u8 dtype (0 f32, 1 f64, 2 i32, 3 i64, 4 u8),
//   u32 ndim, i64 dims[ndim], raw little-endian payload.
// Read back by oracle/mtfa.py.
#pragma once

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

namespace mtfa {

template <typename T> struct code;
template <> struct code<float> { static constexpr uint8_t v = 0; };
template <> struct code<double> { static constexpr uint8_t v = 1; };
template <> struct code<int32_t> { static constexpr uint8_t v = 2; };
template <> struct code<int64_t> { static constexpr uint8_t v = 3; };
template <> struct code<uint8_t> { static constexpr uint8_t v = 4; };

class Writer {
  public:
    explicit Writer(const std::string& path) {
        f_ = std::fopen(path.c_str(), "wb");
        if (!f_) throw std::runtime_error("mtfa: cannot open " + path);
        std::fwrite("MTFA1\n", 1, 6, f_);
    }
    ~Writer() {
        if (f_) std::fclose(f_);
    }
    template <typename T>
    void put(const std::string& name, const std::vector<T>& v, std::vector<int64_t> dims = {}) {
        if (dims.empty()) dims = {static_cast<int64_t>(v.size())};
        int64_t n = 1;
        for (auto d : dims) n *= d;
        if (n != static_cast<int64_t>(v.size())) throw std::runtime_error("mtfa: dims mismatch for " + name);
        uint32_t len = static_cast<uint32_t>(name.size());
        std::fwrite(&len, 4, 1, f_);
        std::fwrite(name.data(), 1, len, f_);
        uint8_t c = code<T>::v;
        std::fwrite(&c, 1, 1, f_);
        uint32_t nd = static_cast<uint32_t>(dims.size());
        std::fwrite(&nd, 4, 1, f_);
        std::fwrite(dims.data(), 8, nd, f_);
        if (!v.empty()) std::fwrite(v.data(), sizeof(T), v.size(), f_);
    }
    void put_str(const std::string& name, const std::string& s) {
        put(name, std::vector<uint8_t>(s.begin(), s.end()));
    }

  private:
    FILE* f_ = nullptr;
};

}  // namespace mtfa
