// HODLR debug serializer: JSON manifest + row-major little-endian float64
// sidecars. Restates the wire format of write_hodlr_debug / read_hodlr_debug
// (reference io.cpp:171-233 and :235-275, declared io.hpp:33-36) on top of the
// device panel form, so a manifest written here is byte-identical to one the
// reference writes for the same matrix (nlohmann dump(2) style: two-space
// indent, keys in sorted order, one array element per line).
//
// The manifest and the sidecars are host artefacts; the device side is one
// panel export (write) or one panel import (read).
#include <algorithm>
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <sstream>

#include "../../include/hodlrgp_b200.h"
#include "api.cuh"
#include "io.cuh"

static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "sidecars are little-endian float64 (io.cpp:13-14)");

namespace hg {

namespace {

namespace fs = std::filesystem;

// ------------------------------------------------------------------ JSON
struct Json {
    enum Kind { Null, Bool, Int, Num, Str, Arr, Obj } kind = Null;
    bool b = false;
    long long i = 0;
    double d = 0.0;
    std::string s;
    std::vector<Json> a;
    std::map<std::string, Json> o;  // sorted keys, as nlohmann::json's default map

    static Json integer(long long v) {
        Json j;
        j.kind = Int;
        j.i = v;
        return j;
    }
    static Json boolean(bool v) {
        Json j;
        j.kind = Bool;
        j.b = v;
        return j;
    }
    static Json str(std::string v) {
        Json j;
        j.kind = Str;
        j.s = std::move(v);
        return j;
    }
    static Json array() {
        Json j;
        j.kind = Arr;
        return j;
    }
    static Json object() {
        Json j;
        j.kind = Obj;
        return j;
    }
    static Json pair(long long x, long long y) {
        Json j = array();
        j.a.push_back(integer(x));
        j.a.push_back(integer(y));
        return j;
    }

    const Json& at(const std::string& key, const std::string& where) const {
        if (kind != Obj) throw IoError(where + ": expected a JSON object");
        auto it = o.find(key);
        if (it == o.end()) throw IoError(where + ": missing key '" + key + "'");
        return it->second;
    }
    long long as_int(const std::string& where) const {
        if (kind == Int) return i;
        if (kind == Num && d == double(static_cast<long long>(d))) return static_cast<long long>(d);
        throw IoError(where + ": expected an integer");
    }
    bool as_bool(const std::string& where) const {
        if (kind != Bool) throw IoError(where + ": expected a boolean");
        return b;
    }
    const std::string& as_str(const std::string& where) const {
        if (kind != Str) throw IoError(where + ": expected a string");
        return s;
    }
    const std::vector<Json>& as_arr(const std::string& where) const {
        if (kind != Arr) throw IoError(where + ": expected an array");
        return a;
    }
};

void escape(std::string& out, const std::string& s) {
    out += '"';
    for (unsigned char c : s) {
        switch (c) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\b': out += "\\b"; break;
            case '\f': out += "\\f"; break;
            case '\n': out += "\\n"; break;
            case '\r': out += "\\r"; break;
            case '\t': out += "\\t"; break;
            default:
                if (c < 0x20) {
                    char buf[8];
                    std::snprintf(buf, sizeof(buf), "\\u%04x", c);
                    out += buf;
                } else {
                    out += char(c);
                }
        }
    }
    out += '"';
}

/// nlohmann::json::dump(2): nested containers one element per line, empty
/// containers as [] / {}, "key": value.
void dump(std::string& out, const Json& j, int depth) {
    const std::string pad(static_cast<size_t>(2 * (depth + 1)), ' '), close(static_cast<size_t>(2 * depth), ' ');
    switch (j.kind) {
        case Json::Null: out += "null"; break;
        case Json::Bool: out += j.b ? "true" : "false"; break;
        case Json::Int: out += std::to_string(j.i); break;
        case Json::Num: {
            char buf[32];
            std::snprintf(buf, sizeof(buf), "%.17g", j.d);
            out += buf;
            break;
        }
        case Json::Str: escape(out, j.s); break;
        case Json::Arr:
            if (j.a.empty()) {
                out += "[]";
                break;
            }
            out += "[\n";
            for (size_t e = 0; e < j.a.size(); ++e) {
                out += pad;
                dump(out, j.a[e], depth + 1);
                out += e + 1 < j.a.size() ? ",\n" : "\n";
            }
            out += close + "]";
            break;
        case Json::Obj: {
            if (j.o.empty()) {
                out += "{}";
                break;
            }
            out += "{\n";
            size_t e = 0;
            for (const auto& kv : j.o) {
                out += pad;
                escape(out, kv.first);
                out += ": ";
                dump(out, kv.second, depth + 1);
                out += ++e < j.o.size() ? ",\n" : "\n";
            }
            out += close + "}";
            break;
        }
    }
}

/// Strict RFC 8259 reader (the subset a manifest can hold; \u escapes are
/// decoded to UTF-8).
class Parser {
public:
    Parser(const std::string& text, std::string where) : t_(text), where_(std::move(where)) {}

    Json document() {
        Json j = value(0);
        ws();
        if (p_ != t_.size()) fail("trailing characters");
        return j;
    }

private:
    const std::string& t_;
    std::string where_;
    size_t p_ = 0;

    [[noreturn]] void fail(const std::string& what) const {
        throw IoError(where_ + ": malformed manifest (" + what + " at byte " + std::to_string(p_) + ")");
    }
    void ws() {
        while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\n' || t_[p_] == '\r' || t_[p_] == '\t')) ++p_;
    }
    bool lit(const char* w) {
        const size_t m = std::strlen(w);
        if (t_.compare(p_, m, w) != 0) return false;
        p_ += m;
        return true;
    }
    Json value(int depth) {
        if (depth > 64) fail("nesting too deep");
        ws();
        if (p_ >= t_.size()) fail("unexpected end");
        const char c = t_[p_];
        if (c == '{') return object(depth);
        if (c == '[') return array(depth);
        if (c == '"') return Json::str(string());
        if (lit("true")) return Json::boolean(true);
        if (lit("false")) return Json::boolean(false);
        if (lit("null")) return Json{};
        return number();
    }
    Json object(int depth) {
        Json j = Json::object();
        ++p_;
        ws();
        if (p_ < t_.size() && t_[p_] == '}') {
            ++p_;
            return j;
        }
        for (;;) {
            ws();
            if (p_ >= t_.size() || t_[p_] != '"') fail("expected a key");
            std::string k = string();
            ws();
            if (p_ >= t_.size() || t_[p_] != ':') fail("expected ':'");
            ++p_;
            j.o[k] = value(depth + 1);
            ws();
            if (p_ < t_.size() && t_[p_] == ',') {
                ++p_;
                continue;
            }
            if (p_ < t_.size() && t_[p_] == '}') {
                ++p_;
                return j;
            }
            fail("expected ',' or '}'");
        }
    }
    Json array(int depth) {
        Json j = Json::array();
        ++p_;
        ws();
        if (p_ < t_.size() && t_[p_] == ']') {
            ++p_;
            return j;
        }
        for (;;) {
            j.a.push_back(value(depth + 1));
            ws();
            if (p_ < t_.size() && t_[p_] == ',') {
                ++p_;
                continue;
            }
            if (p_ < t_.size() && t_[p_] == ']') {
                ++p_;
                return j;
            }
            fail("expected ',' or ']'");
        }
    }
    static void utf8(std::string& out, unsigned cp) {
        if (cp < 0x80) {
            out += char(cp);
        } else if (cp < 0x800) {
            out += char(0xC0 | (cp >> 6));
            out += char(0x80 | (cp & 0x3F));
        } else if (cp < 0x10000) {
            out += char(0xE0 | (cp >> 12));
            out += char(0x80 | ((cp >> 6) & 0x3F));
            out += char(0x80 | (cp & 0x3F));
        } else {
            out += char(0xF0 | (cp >> 18));
            out += char(0x80 | ((cp >> 12) & 0x3F));
            out += char(0x80 | ((cp >> 6) & 0x3F));
            out += char(0x80 | (cp & 0x3F));
        }
    }
    unsigned hex4() {
        if (p_ + 4 > t_.size()) fail("short \\u escape");
        unsigned v = 0;
        for (int e = 0; e < 4; ++e) {
            const char c = t_[p_++];
            v <<= 4;
            if (c >= '0' && c <= '9') v |= unsigned(c - '0');
            else if (c >= 'a' && c <= 'f') v |= unsigned(c - 'a' + 10);
            else if (c >= 'A' && c <= 'F') v |= unsigned(c - 'A' + 10);
            else fail("bad \\u escape");
        }
        return v;
    }
    std::string string() {
        std::string out;
        ++p_;  // opening quote
        for (;;) {
            if (p_ >= t_.size()) fail("unterminated string");
            const unsigned char c = static_cast<unsigned char>(t_[p_++]);
            if (c == '"') return out;
            if (c < 0x20) fail("control character in string");
            if (c != '\\') {
                out += char(c);
                continue;
            }
            if (p_ >= t_.size()) fail("unterminated escape");
            const char e = t_[p_++];
            switch (e) {
                case '"': out += '"'; break;
                case '\\': out += '\\'; break;
                case '/': out += '/'; break;
                case 'b': out += '\b'; break;
                case 'f': out += '\f'; break;
                case 'n': out += '\n'; break;
                case 'r': out += '\r'; break;
                case 't': out += '\t'; break;
                case 'u': {
                    unsigned cp = hex4();
                    if (cp >= 0xD800 && cp < 0xDC00) {
                        if (!lit("\\u")) fail("lone surrogate");
                        const unsigned lo = hex4();
                        if (lo < 0xDC00 || lo >= 0xE000) fail("bad surrogate pair");
                        cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                    }
                    utf8(out, cp);
                    break;
                }
                default: fail("bad escape");
            }
        }
    }
    Json number() {
        const size_t start = p_;
        if (p_ < t_.size() && t_[p_] == '-') ++p_;
        bool integral = true;
        auto digits = [&] {
            const size_t s0 = p_;
            while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
            if (p_ == s0) fail("expected a digit");
        };
        digits();
        if (p_ < t_.size() && t_[p_] == '.') {
            ++p_;
            integral = false;
            digits();
        }
        if (p_ < t_.size() && (t_[p_] == 'e' || t_[p_] == 'E')) {
            ++p_;
            integral = false;
            if (p_ < t_.size() && (t_[p_] == '+' || t_[p_] == '-')) ++p_;
            digits();
        }
        const std::string tok = t_.substr(start, p_ - start);
        Json j;
        if (integral) {
            errno = 0;
            char* end = nullptr;
            const long long v = std::strtoll(tok.c_str(), &end, 10);
            if (errno == 0 && end && *end == '\0') return Json::integer(v);
        }
        j.kind = Json::Num;
        j.d = std::strtod(tok.c_str(), nullptr);
        return j;
    }
};

// -------------------------------------------------------------- sidecars
/// io.cpp:78-87: row-major float64. `src(i, c)` gives element (i, c).
template <class F>
void write_sidecar(const fs::path& path, i64 rows, i64 cols, F&& src) {
    std::vector<double> buf(static_cast<size_t>(rows) * static_cast<size_t>(cols));
    for (i64 i = 0; i < rows; ++i)
        for (i64 c = 0; c < cols; ++c) buf[static_cast<size_t>(i * cols + c)] = src(i, c);
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot write " + path.string());
    out.write(reinterpret_cast<const char*>(buf.data()), std::streamsize(buf.size() * sizeof(double)));
    if (!out) throw IoError("cannot write " + path.string());
}

/// io.cpp:89-101: rows x cols row-major; fewer bytes than that is an error,
/// trailing bytes are ignored.
template <class F>
void read_sidecar(const fs::path& path, i64 rows, i64 cols, F&& dst) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open " + path.string());
    std::vector<double> buf(static_cast<size_t>(rows) * static_cast<size_t>(cols));
    in.read(reinterpret_cast<char*>(buf.data()), std::streamsize(buf.size() * sizeof(double)));
    if (!in) throw IoError(path.string() + ": truncated sidecar");
    for (i64 i = 0; i < rows; ++i)
        for (i64 c = 0; c < cols; ++c) dst(i, c, buf[static_cast<size_t>(i * cols + c)]);
}

/// Where block (l, j) of one triangle sits in the panel form (hodlr.cuh):
/// upper = U_l[left child] V_l[right child]^T, lower = U_l[right] V_l[left]^T.
struct BlockPlace {
    Range rows, cols;
};
BlockPlace place(const ClusterTree& t, int l, i64 j, bool upper) {
    const Range a = t.level(l)[static_cast<size_t>(2 * j)], b = t.level(l)[static_cast<size_t>(2 * j + 1)];
    return upper ? BlockPlace{a, b} : BlockPlace{b, a};
}

std::string block_base(const std::string& name, const char* tag, int l, i64 j) {
    return name + "_" + tag + "_l" + std::to_string(l) + "_n" + std::to_string(j);
}

}  // namespace

// io.cpp:171-233
void write_hodlr_debug(const std::string& dir, const std::string& name, const DHodlr& h) {
    const ClusterTree& t = h.tree->host;
    const i64 n = h.n();
    const int tau = h.tau();
    std::vector<double> flat(h.export_size());
    const size_t nodes = std::max<size_t>((size_t(1) << tau) - 1, 1);
    std::vector<int> ru(nodes, 0), rl(nodes, 0);
    h.export_panels(flat.data(), ru.data(), rl.data());  // synchronizes
    std::error_code ec;
    fs::create_directories(dir, ec);
    if (ec) throw IoError("cannot create " + dir + ": " + ec.message());
    const fs::path root(dir);

    // Panel offsets per level: U_l at off[l-1], V_l right after it.
    std::vector<size_t> off(static_cast<size_t>(tau) + 1, 0);
    for (int l = 1; l <= tau; ++l)
        off[static_cast<size_t>(l)] = off[static_cast<size_t>(l - 1)] + 2 * static_cast<size_t>(n) * static_cast<size_t>(h.Rl(l));

    Json m = Json::object();
    m.o["n"] = Json::integer(n);
    m.o["depth"] = Json::integer(tau);
    m.o["symmetric"] = Json::boolean(h.sym);
    auto triangle = [&](bool upper) {
        Json levels = Json::array();
        size_t node = 0;
        for (int l = 1; l <= tau; ++l) {
            const double* U = flat.data() + off[static_cast<size_t>(l - 1)];
            const double* V = U + static_cast<size_t>(n) * static_cast<size_t>(h.Rl(l));
            Json lev = Json::object();
            lev.o["level"] = Json::integer(l);
            Json blocks = Json::array();
            const i64 cnt = i64(t.level(l - 1).size());
            for (i64 j = 0; j < cnt; ++j, ++node) {
                const BlockPlace bp = place(t, l, j, upper);
                const int r = upper ? ru[node] : rl[node];
                const std::string base = block_base(name, upper ? "u" : "lo", l, j);
                Json e = Json::object();
                e.o["node"] = Json::integer(j);
                e.o["rows"] = Json::pair(bp.rows.lo, bp.rows.hi);
                e.o["cols"] = Json::pair(bp.cols.lo, bp.cols.hi);
                e.o["rank"] = Json::integer(r);
                e.o["left"] = Json::str(base + "_left.bin");
                e.o["right"] = Json::str(base + "_right.bin");
                write_sidecar(root / (base + "_left.bin"), bp.rows.size(), r,
                              [&](i64 i, i64 c) { return U[static_cast<size_t>(bp.rows.lo + i + c * n)]; });
                write_sidecar(root / (base + "_right.bin"), bp.cols.size(), r,
                              [&](i64 i, i64 c) { return V[static_cast<size_t>(bp.cols.lo + i + c * n)]; });
                blocks.a.push_back(std::move(e));
            }
            lev.o["blocks"] = std::move(blocks);
            levels.a.push_back(std::move(lev));
        }
        return levels;
    };
    m.o["upper"] = triangle(true);
    if (!h.sym) m.o["lower"] = triangle(false);

    Json leaves = Json::array();
    size_t loff = off[static_cast<size_t>(tau)];
    const auto& lv = t.leaves();
    for (size_t b = 0; b < lv.size(); ++b) {
        const i64 mb = lv[b].size();
        const std::string file = name + "_leaf" + std::to_string(b) + ".bin";
        Json e = Json::object();
        e.o["index"] = Json::integer(i64(b));
        e.o["rows"] = Json::pair(lv[b].lo, lv[b].hi);
        e.o["file"] = Json::str(file);
        const double* L = flat.data() + loff;
        write_sidecar(root / file, mb, mb, [&](i64 i, i64 c) { return L[static_cast<size_t>(i + c * mb)]; });
        loff += static_cast<size_t>(mb) * static_cast<size_t>(mb);
        leaves.a.push_back(std::move(e));
    }
    m.o["leaves"] = std::move(leaves);

    std::string text;
    dump(text, m, 0);
    text += "\n";
    std::ofstream out(root / (name + ".json"), std::ios::binary);
    if (!out) throw IoError("cannot write manifest in " + dir);
    out << text;
    if (!out) throw IoError("cannot write manifest in " + dir);
}

// io.cpp:235-275
DHodlr read_hodlr_debug(const std::string& dir, const std::string& name) {
    const fs::path root(dir);
    const fs::path mpath = root / (name + ".json");
    std::ifstream in(mpath, std::ios::binary);
    if (!in) throw IoError("cannot open manifest in " + dir);
    std::stringstream ss;
    ss << in.rdbuf();
    const std::string text = ss.str();
    const std::string where = mpath.string();
    const Json m = Parser(text, where).document();

    const long long n = m.at("n", where).as_int(where + " n");
    const long long depth = m.at("depth", where).as_int(where + " depth");
    const bool sym = m.at("symmetric", where).as_bool(where + " symmetric");
    if (n < 1 || depth < 0 || depth > 30 || (n >> depth) < 1)
        throw std::invalid_argument(where + ": n and depth do not describe a cluster tree");
    DTreeP tree = get_tree(n, int(depth));
    const ClusterTree& t = tree->host;
    const int tau = int(depth);

    // Pass 1: per-block ranks (blocks absent from the manifest stay empty,
    // as HodlrMatrix::zero leaves them).
    const size_t nodes = std::max<size_t>((size_t(1) << tau) - 1, 1);
    std::vector<int> ru(nodes, 0), rl(nodes, 0);
    struct Entry {
        int l;
        i64 j;
        bool upper;
        const Json* e;
    };
    std::vector<Entry> entries;
    auto scan = [&](const char* key, bool upper) {
        for (const Json& lev : m.at(key, where).as_arr(where + " " + key)) {
            const long long l = lev.at("level", where).as_int(where + " level");
            if (l < 1 || l > tau) throw std::invalid_argument(where + ": level " + std::to_string(l) + " out of range");
            for (const Json& e : lev.at("blocks", where).as_arr(where + " blocks")) {
                const long long j = e.at("node", where).as_int(where + " node");
                if (j < 0 || j >= (1LL << (l - 1)))
                    throw std::invalid_argument(where + ": node " + std::to_string(j) + " out of range");
                const BlockPlace bp = place(t, int(l), j, upper);
                const auto& rows = e.at("rows", where).as_arr(where + " rows");
                const auto& cols = e.at("cols", where).as_arr(where + " cols");
                if (rows.size() != 2 || cols.size() != 2 || rows[0].as_int(where) != bp.rows.lo ||
                    rows[1].as_int(where) != bp.rows.hi || cols[0].as_int(where) != bp.cols.lo ||
                    cols[1].as_int(where) != bp.cols.hi)
                    throw std::invalid_argument(where + ": block ranges do not match the cluster tree");
                const long long r = e.at("rank", where).as_int(where + " rank");
                if (r < 0 || r > (1LL << 30)) throw std::invalid_argument(where + ": negative rank");
                const size_t idx = (size_t(1) << (l - 1)) - 1 + size_t(j);
                (upper ? ru : rl)[idx] = int(r);
                entries.push_back(Entry{int(l), j, upper, &e});
            }
        }
    };
    scan("upper", true);
    if (!sym) scan("lower", false);

    std::vector<int> R(static_cast<size_t>(std::max(tau, 1)), 0);
    for (int l = 1; l <= tau; ++l)
        for (i64 j = 0; j < (i64(1) << (l - 1)); ++j) {
            const size_t idx = (size_t(1) << (l - 1)) - 1 + size_t(j);
            R[static_cast<size_t>(l - 1)] = std::max({R[static_cast<size_t>(l - 1)], ru[idx], sym ? 0 : rl[idx]});
        }
    std::vector<size_t> off(static_cast<size_t>(tau) + 1, 0);
    for (int l = 1; l <= tau; ++l)
        off[static_cast<size_t>(l)] = off[static_cast<size_t>(l - 1)] + 2 * static_cast<size_t>(n) * static_cast<size_t>(R[static_cast<size_t>(l - 1)]);
    size_t total = off[static_cast<size_t>(tau)];
    for (const Range& r : t.leaves()) total += static_cast<size_t>(r.size()) * static_cast<size_t>(r.size());
    std::vector<double> flat(total, 0.0);

    // Pass 2: sidecars into the panels.
    for (const Entry& en : entries) {
        const BlockPlace bp = place(t, en.l, en.j, en.upper);
        const size_t Rl = static_cast<size_t>(R[static_cast<size_t>(en.l - 1)]);
        double* U = flat.data() + off[static_cast<size_t>(en.l - 1)];
        // Symmetric panels keep V_l == U_l (hodlr.cuh): upper.right lands in
        // U_l's rows of the right child, which also spell the lower blocks.
        double* V = sym ? U : U + static_cast<size_t>(n) * Rl;
        const int r = (en.upper ? ru : rl)[(size_t(1) << (en.l - 1)) - 1 + size_t(en.j)];
        read_sidecar(root / en.e->at("left", where).as_str(where + " left"), bp.rows.size(), r,
                     [&](i64 i, i64 c, double v) { U[static_cast<size_t>(bp.rows.lo + i + c * n)] = v; });
        read_sidecar(root / en.e->at("right", where).as_str(where + " right"), bp.cols.size(), r,
                     [&](i64 i, i64 c, double v) { V[static_cast<size_t>(bp.cols.lo + i + c * n)] = v; });
    }
    std::vector<size_t> leaf_off(t.leaves().size(), 0);
    {
        size_t o = off[static_cast<size_t>(tau)];
        for (size_t b = 0; b < t.leaves().size(); ++b) {
            leaf_off[b] = o;
            o += static_cast<size_t>(t.leaves()[b].size()) * static_cast<size_t>(t.leaves()[b].size());
        }
    }
    for (const Json& e : m.at("leaves", where).as_arr(where + " leaves")) {
        const long long b = e.at("index", where).as_int(where + " index");
        if (b < 0 || b >= (long long)t.leaves().size())
            throw std::invalid_argument(where + ": leaf index " + std::to_string(b) + " out of range");
        const Range lr = t.leaves()[static_cast<size_t>(b)];
        const auto& rows = e.at("rows", where).as_arr(where + " rows");
        if (rows.size() != 2 || rows[0].as_int(where) != lr.lo || rows[1].as_int(where) != lr.hi)
            throw std::invalid_argument(where + ": leaf ranges do not match the cluster tree");
        const i64 mb = lr.size();
        double* L = flat.data() + leaf_off[static_cast<size_t>(b)];
        read_sidecar(root / e.at("file", where).as_str(where + " file"), mb, mb,
                     [&](i64 i, i64 c, double v) { L[static_cast<size_t>(i + c * mb)] = v; });
    }
    return DHodlr::import_panels(tree, sym, R.data(), flat.data(), ru.data(), rl.data());
}

}  // namespace hg
