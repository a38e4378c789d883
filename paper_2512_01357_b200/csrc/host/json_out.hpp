// Tiny append-only JSON writer for pool dumps (no third-party dependency).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>

namespace tg {

class JsonOut {
public:
    void raw(const char* s) { s_ += s; }
    void str(const std::string& v) {
        s_ += '"';
        for (char c : v) {
            const unsigned char u = static_cast<unsigned char>(c);
            if (c == '"' || c == '\\') {
                s_ += '\\';
                s_ += c;
            } else if (u < 0x20) {
                char buf[8];
                std::snprintf(buf, sizeof buf, "\\u%04x", u);
                s_ += buf;
            } else {
                s_ += c;
            }
        }
        s_ += '"';
    }
    void num(std::uint64_t v) { s_ += std::to_string(v); }
    // Shortest round-trip representation; integral values keep a ".0" like
    // nlohmann::json so dumps parse to the same typed values.
    void dbl(double v) {
        if (!std::isfinite(v)) {
            s_ += "null";
            return;
        }
        char buf[40];
        for (int prec = 1; prec <= 17; ++prec) {
            std::snprintf(buf, sizeof buf, "%.*g", prec, v);
            if (std::strtod(buf, nullptr) == v) break;
        }
        std::string t = buf;
        if (t.find_first_of(".eEn") == std::string::npos) t += ".0";
        s_ += t;
    }
    std::string take() { return std::move(s_); }

private:
    std::string s_;
};

}  // namespace tg
