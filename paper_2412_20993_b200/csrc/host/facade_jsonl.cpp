// facade_jsonl.cpp — probe trace JSON-lines I/O (probe.cpp:126-182):
// the host-side input boundary that turns recorded traces into the answer arena.
//
// The reference parses each line with nlohmann::json (an un-vendored third-party library,
// SURVEY.md §8(c)); this is a self-contained RFC 8259 reader that follows the same
// acceptance rules for the five fields: numbers convert to int/long the way nlohmann's
// get<>() casts them (integers wrap, floats truncate), strings must be valid UTF-8 with
// no raw control bytes, duplicate keys keep the last value, trailing bytes are an error.
// Errors keep the reference's message structure — "trace line <n>: invalid JSON: …",
// "trace line <n>: missing or mistyped field: …", "trace line <n>: token_offset does not
// increase" / "step_index does not increase" — the detail after the category names the
// problem in this parser's words, not nlohmann's exception text.  Writing emits nlohmann's
// compact dump() layout (keys in std::map order, same escapes).

#include <cerrno>
#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <istream>
#include <map>
#include <ostream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "cdx/metrics.hpp"
#include "cdx/probe.hpp"

namespace cdx::probe {

namespace {

struct JsonError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct FieldError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct Value {
    enum Kind { Null, Bool, Int, Uint, Float, String, Array, Object } kind = Null;
    bool b = false;
    int64_t i = 0;
    uint64_t u = 0;
    double d = 0.0;
    std::string s;
    std::vector<Value> arr;
    std::vector<std::pair<std::string, Value>> obj;

    const Value* find(const std::string& k) const {
        const Value* hit = nullptr;
        for (const auto& kv : obj)
            if (kv.first == k) hit = &kv.second;  // last duplicate wins
        return hit;
    }
};

const char* kind_name(Value::Kind k) {
    switch (k) {
        case Value::Null: return "null";
        case Value::Bool: return "boolean";
        case Value::Int:
        case Value::Uint:
        case Value::Float: return "number";
        case Value::String: return "string";
        case Value::Array: return "array";
        case Value::Object: return "object";
    }
    return "?";
}

class Reader {
public:
    explicit Reader(const std::string& t) : t_(t) {}

    Value document() {
        ws();
        Value v = value(0);
        ws();
        if (p_ != t_.size()) fail("unexpected trailing characters");
        return v;
    }

private:
    [[noreturn]] void fail(const std::string& what) const {
        throw JsonError("syntax error at byte " + std::to_string(p_ + 1) + ": " + what);
    }
    void ws() {
        while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\t' || t_[p_] == '\n' || t_[p_] == '\r')) ++p_;
    }
    bool eat(char c) {
        if (p_ < t_.size() && t_[p_] == c) {
            ++p_;
            return true;
        }
        return false;
    }
    void literal(const char* w) {
        for (const char* c = w; *c; ++c)
            if (!eat(*c)) fail(std::string("invalid literal, expected '") + w + "'");
    }
    Value value(int depth) {
        if (depth > 512) fail("nesting too deep");
        if (p_ >= t_.size()) fail("unexpected end of input");
        Value v;
        const char c = t_[p_];
        if (c == '{') {
            ++p_;
            v.kind = Value::Object;
            ws();
            if (eat('}')) return v;
            for (;;) {
                ws();
                if (p_ >= t_.size() || t_[p_] != '"') fail("expected a string object key");
                std::string k = string_lit();
                ws();
                if (!eat(':')) fail("expected ':'");
                ws();
                Value x = value(depth + 1);
                v.obj.emplace_back(std::move(k), std::move(x));
                ws();
                if (eat(',')) continue;
                if (eat('}')) return v;
                fail("expected ',' or '}'");
            }
        }
        if (c == '[') {
            ++p_;
            v.kind = Value::Array;
            ws();
            if (eat(']')) return v;
            for (;;) {
                ws();
                v.arr.push_back(value(depth + 1));
                ws();
                if (eat(',')) continue;
                if (eat(']')) return v;
                fail("expected ',' or ']'");
            }
        }
        if (c == '"') {
            v.kind = Value::String;
            v.s = string_lit();
            return v;
        }
        if (c == 't') {
            literal("true");
            v.kind = Value::Bool;
            v.b = true;
            return v;
        }
        if (c == 'f') {
            literal("false");
            v.kind = Value::Bool;
            return v;
        }
        if (c == 'n') {
            literal("null");
            return v;
        }
        if (c == '-' || (c >= '0' && c <= '9')) return number();
        fail("unexpected character");
    }
    Value number() {
        const size_t b = p_;
        const bool neg = eat('-');
        if (p_ >= t_.size() || !(t_[p_] >= '0' && t_[p_] <= '9')) fail("invalid number");
        if (t_[p_] == '0') {
            ++p_;
            if (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') fail("leading zero in number");
        } else {
            while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
        }
        bool is_float = false;
        if (eat('.')) {
            is_float = true;
            if (p_ >= t_.size() || !(t_[p_] >= '0' && t_[p_] <= '9')) fail("invalid number fraction");
            while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
        }
        if (p_ < t_.size() && (t_[p_] == 'e' || t_[p_] == 'E')) {
            is_float = true;
            ++p_;
            if (!eat('+')) eat('-');
            if (p_ >= t_.size() || !(t_[p_] >= '0' && t_[p_] <= '9')) fail("invalid number exponent");
            while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
        }
        const std::string tok = t_.substr(b, p_ - b);
        Value v;
        if (!is_float) {
            errno = 0;
            if (neg) {
                char* end = nullptr;
                const long long x = std::strtoll(tok.c_str(), &end, 10);
                if (errno == 0) {
                    v.kind = Value::Int;
                    v.i = x;
                    return v;
                }
            } else {
                char* end = nullptr;
                const unsigned long long x = std::strtoull(tok.c_str(), &end, 10);
                if (errno == 0) {
                    v.kind = Value::Uint;
                    v.u = x;
                    return v;
                }
            }
        }
        v.kind = Value::Float;
        v.d = std::strtod(tok.c_str(), nullptr);
        if (!std::isfinite(v.d)) fail("number out of range");
        return v;
    }
    static void put_utf8(std::string& o, uint32_t cp) {
        if (cp < 0x80) {
            o += static_cast<char>(cp);
        } else if (cp < 0x800) {
            o += static_cast<char>(0xC0 | (cp >> 6));
            o += static_cast<char>(0x80 | (cp & 0x3F));
        } else if (cp < 0x10000) {
            o += static_cast<char>(0xE0 | (cp >> 12));
            o += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
            o += static_cast<char>(0x80 | (cp & 0x3F));
        } else {
            o += static_cast<char>(0xF0 | (cp >> 18));
            o += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
            o += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
            o += static_cast<char>(0x80 | (cp & 0x3F));
        }
    }
    uint32_t hex4() {
        if (p_ + 4 > t_.size()) fail("truncated \\u escape");
        uint32_t v = 0;
        for (int k = 0; k < 4; ++k) {
            const char c = t_[p_++];
            v <<= 4;
            if (c >= '0' && c <= '9') v |= static_cast<uint32_t>(c - '0');
            else if (c >= 'a' && c <= 'f') v |= static_cast<uint32_t>(c - 'a' + 10);
            else if (c >= 'A' && c <= 'F') v |= static_cast<uint32_t>(c - 'A' + 10);
            else fail("invalid \\u escape");
        }
        return v;
    }
    std::string string_lit() {
        ++p_;  // opening quote
        std::string o;
        for (;;) {
            if (p_ >= t_.size()) fail("unterminated string");
            const unsigned char c = static_cast<unsigned char>(t_[p_]);
            if (c == '"') {
                ++p_;
                return o;
            }
            if (c < 0x20) fail("control character in string must be escaped");
            if (c == '\\') {
                ++p_;
                if (p_ >= t_.size()) fail("unterminated escape");
                const char e = t_[p_++];
                switch (e) {
                    case '"': o += '"'; break;
                    case '\\': o += '\\'; break;
                    case '/': o += '/'; break;
                    case 'b': o += '\b'; break;
                    case 'f': o += '\f'; break;
                    case 'n': o += '\n'; break;
                    case 'r': o += '\r'; break;
                    case 't': o += '\t'; break;
                    case 'u': {
                        uint32_t cp = hex4();
                        if (cp >= 0xD800 && cp <= 0xDBFF) {
                            if (!(eat('\\') && eat('u'))) fail("unpaired surrogate");
                            const uint32_t lo = hex4();
                            if (lo < 0xDC00 || lo > 0xDFFF) fail("unpaired surrogate");
                            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                        } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
                            fail("unpaired surrogate");
                        }
                        put_utf8(o, cp);
                        break;
                    }
                    default: fail("invalid escape");
                }
                continue;
            }
            // raw UTF-8 sequence: validate (overlongs, surrogates, > U+10FFFF rejected)
            int len = 0;
            uint32_t cp = 0;
            if (c < 0x80) len = 1, cp = c;
            else if (c >= 0xC2 && c <= 0xDF) len = 2, cp = c & 0x1F;
            else if (c >= 0xE0 && c <= 0xEF) len = 3, cp = c & 0x0F;
            else if (c >= 0xF0 && c <= 0xF4) len = 4, cp = c & 0x07;
            else fail("invalid UTF-8 byte");
            if (p_ + len > t_.size()) fail("truncated UTF-8 sequence");
            for (int k = 1; k < len; ++k) {
                const unsigned char cc = static_cast<unsigned char>(t_[p_ + k]);
                if ((cc & 0xC0) != 0x80) fail("invalid UTF-8 continuation");
                cp = (cp << 6) | (cc & 0x3F);
            }
            if ((len == 3 && (cp < 0x800 || (cp >= 0xD800 && cp <= 0xDFFF))) || (len == 4 && (cp < 0x10000 || cp > 0x10FFFF)))
                fail("invalid UTF-8 sequence");
            o.append(t_, p_, static_cast<size_t>(len));
            p_ += static_cast<size_t>(len);
        }
    }

    const std::string& t_;
    size_t p_ = 0;
};

const Value& at(const Value& j, const char* key) {
    if (j.kind != Value::Object)
        throw FieldError(std::string("cannot use at() with ") + kind_name(j.kind));
    const Value* v = j.find(key);
    if (!v) throw FieldError(std::string("key '") + key + "' not found");
    return *v;
}

// nlohmann get<int>() (the generic arithmetic overload) also converts booleans; get<long>()
// (= number_integer_t on LP64) does not.
template <class I>
I as_integer(const Value& v, const char* key, bool allow_bool) {
    switch (v.kind) {
        case Value::Int: return static_cast<I>(v.i);
        case Value::Uint: return static_cast<I>(v.u);
        case Value::Float: return static_cast<I>(v.d);
        case Value::Bool:
            if (allow_bool) return static_cast<I>(v.b);
            [[fallthrough]];
        default: throw FieldError(std::string(key) + ": type must be number, but is " + kind_name(v.kind));
    }
}

std::string as_string(const Value& v, const char* key) {
    if (v.kind != Value::String)
        throw FieldError(std::string(key) + ": type must be string, but is " + kind_name(v.kind));
    return v.s;
}

void dump_string(std::ostream& out, const std::string& s) {
    out << '"';
    for (unsigned char c : s) {
        switch (c) {
            case '"': out << "\\\""; break;
            case '\\': out << "\\\\"; break;
            case '\b': out << "\\b"; break;
            case '\f': out << "\\f"; break;
            case '\n': out << "\\n"; break;
            case '\r': out << "\\r"; break;
            case '\t': out << "\\t"; break;
            default:
                if (c < 0x20) {
                    char buf[8];
                    std::snprintf(buf, sizeof buf, "\\u%04x", c);
                    out << buf;
                } else {
                    out << static_cast<char>(c);
                }
        }
    }
    out << '"';
}

}  // namespace

std::vector<TraceLine> read_trace_jsonl(std::istream& in) {
    std::vector<TraceLine> out;
    std::map<std::string, std::pair<long, int>> last;  // program -> (offset, step)
    std::string line;
    long line_no = 0;
    while (std::getline(in, line)) {
        ++line_no;
        if (metrics::trim(line).empty()) continue;
        const std::string where = "trace line " + std::to_string(line_no) + ": ";
        Value j;
        try {
            j = Reader(line).document();
        } catch (const JsonError& e) {
            throw std::runtime_error(where + "invalid JSON: " + e.what());
        }
        TraceLine t;
        try {
            t.program_id = as_string(at(j, "program_id"), "program_id");
            t.record.step_index = as_integer<int>(at(j, "step_index"), "step_index", true);
            t.record.token_offset = as_integer<long>(at(j, "token_offset"), "token_offset", false);
            t.record.answer = as_string(at(j, "answer"), "answer");
            const Value* h = j.find("hesitant");
            if (h) {
                if (h->kind != Value::Bool)
                    throw FieldError(std::string("hesitant: type must be boolean, but is ") + kind_name(h->kind));
                t.record.hesitant = h->b;
            }
        } catch (const FieldError& e) {
            throw std::runtime_error(where + "missing or mistyped field: " + e.what());
        }
        auto it = last.find(t.program_id);
        if (it != last.end()) {
            if (t.record.token_offset <= it->second.first)
                throw std::runtime_error(where + "token_offset does not increase");
            if (t.record.step_index <= it->second.second)
                throw std::runtime_error(where + "step_index does not increase");
        }
        last[t.program_id] = {t.record.token_offset, t.record.step_index};
        out.push_back(std::move(t));
    }
    return out;
}

std::vector<TraceLine> read_trace_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open trace file: " + path);
    return read_trace_jsonl(in);
}

void write_trace_jsonl(std::ostream& out, std::span<const TraceLine> lines) {
    for (const auto& t : lines) {
        out << "{\"answer\":";
        dump_string(out, t.record.answer);
        out << ",\"hesitant\":" << (t.record.hesitant ? "true" : "false") << ",\"program_id\":";
        dump_string(out, t.program_id);
        out << ",\"step_index\":" << t.record.step_index << ",\"token_offset\":" << t.record.token_offset << "}\n";
    }
}

}  // namespace cdx::probe
