// json.hpp -- minimal JSON document model for the graph IR (internal to librf_fa.so).
//
// The reference reads and writes its graph files with an un-vendored third-party JSON library
// (proj/core/src/graph.cpp:13); this build has no third-party code, so the little JSON the IR
// needs is implemented here: a recursive-descent parser that keeps integers and reals apart
// (the IR's attribute typing depends on it, graph.cpp:109-131), insertion-ordered objects, and
// a pretty printer whose output format (2-space indent, one array element per line, shortest
// round-trip reals that always carry a fraction or an exponent) is byte-compatible with what the
// reference's serialize_graph emits (graph.cpp:195-230), so that rewritten graphs can be diffed
// against the reference's as text.
#pragma once

#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

namespace rfjson {

struct ParseError {
    std::string what;
};

class Value {
public:
    enum class Kind { Null, Bool, Int, Real, String, Array, Object };
    using Member = std::pair<std::string, Value>;

    Value() = default;
    static Value integer(int64_t v) {
        Value x;
        x.kind_ = Kind::Int;
        x.int_ = v;
        return x;
    }
    static Value real(double v) {
        Value x;
        x.kind_ = Kind::Real;
        x.real_ = v;
        return x;
    }
    static Value boolean(bool v) {
        Value x;
        x.kind_ = Kind::Bool;
        x.int_ = v ? 1 : 0;
        return x;
    }
    static Value string(std::string v) {
        Value x;
        x.kind_ = Kind::String;
        x.str_ = std::move(v);
        return x;
    }
    static Value array() {
        Value x;
        x.kind_ = Kind::Array;
        return x;
    }
    static Value object() {
        Value x;
        x.kind_ = Kind::Object;
        return x;
    }

    Kind kind() const { return kind_; }
    bool is_int() const { return kind_ == Kind::Int; }
    bool is_number() const { return kind_ == Kind::Int || kind_ == Kind::Real; }
    bool is_string() const { return kind_ == Kind::String; }
    bool is_array() const { return kind_ == Kind::Array; }
    bool is_object() const { return kind_ == Kind::Object; }

    int64_t as_int() const { return kind_ == Kind::Int ? int_ : static_cast<int64_t>(real_); }
    double as_real() const { return kind_ == Kind::Real ? real_ : static_cast<double>(int_); }
    const std::string& as_string() const { return str_; }
    const std::vector<Value>& items() const { return items_; }
    const std::vector<Member>& members() const { return members_; }

    void push(Value v) { items_.push_back(std::move(v)); }
    void set(std::string key, Value v) { members_.emplace_back(std::move(key), std::move(v)); }
    const Value* find(std::string_view key) const {
        for (const auto& m : members_)
            if (m.first == key) return &m.second;
        return nullptr;
    }

private:
    Kind kind_ = Kind::Null;
    int64_t int_ = 0;
    double real_ = 0.0;
    std::string str_;
    std::vector<Value> items_;
    std::vector<Member> members_;
};

// ---------------------------------------------------------------------------------------------
// parser
// ---------------------------------------------------------------------------------------------
class Parser {
public:
    explicit Parser(std::string_view text) : s_(text) {}

    Value parse_document() {
        Value v = parse_value(0);
        skip_ws();
        if (pos_ != s_.size()) fail("trailing characters");
        return v;
    }

private:
    std::string_view s_;
    size_t pos_ = 0;

    [[noreturn]] void fail(const char* msg) const { throw ParseError{std::string(msg) + " at offset " + std::to_string(pos_)}; }
    void skip_ws() {
        while (pos_ < s_.size() && (s_[pos_] == ' ' || s_[pos_] == '\n' || s_[pos_] == '\t' || s_[pos_] == '\r')) ++pos_;
    }
    bool eat(char c) {
        if (pos_ < s_.size() && s_[pos_] == c) {
            ++pos_;
            return true;
        }
        return false;
    }
    void expect_word(const char* w) {
        const size_t n = std::strlen(w);
        if (s_.substr(pos_, n) != w) fail("bad literal");
        pos_ += n;
    }

    Value parse_value(int depth) {
        if (depth > 256) fail("nesting too deep");
        skip_ws();
        if (pos_ >= s_.size()) fail("unexpected end");
        const char c = s_[pos_];
        if (c == '{') return parse_object(depth);
        if (c == '[') return parse_array(depth);
        if (c == '"') return Value::string(parse_string());
        if (c == 't') {
            expect_word("true");
            return Value::boolean(true);
        }
        if (c == 'f') {
            expect_word("false");
            return Value::boolean(false);
        }
        if (c == 'n') {
            expect_word("null");
            return Value();
        }
        return parse_number();
    }

    Value parse_object(int depth) {
        Value obj = Value::object();
        ++pos_;  // {
        skip_ws();
        if (eat('}')) return obj;
        for (;;) {
            skip_ws();
            if (pos_ >= s_.size() || s_[pos_] != '"') fail("object key must be a string");
            std::string key = parse_string();
            skip_ws();
            if (!eat(':')) fail("expected ':'");
            obj.set(std::move(key), parse_value(depth + 1));
            skip_ws();
            if (eat(',')) continue;
            if (eat('}')) return obj;
            fail("expected ',' or '}'");
        }
    }

    Value parse_array(int depth) {
        Value arr = Value::array();
        ++pos_;  // [
        skip_ws();
        if (eat(']')) return arr;
        for (;;) {
            arr.push(parse_value(depth + 1));
            skip_ws();
            if (eat(',')) continue;
            if (eat(']')) return arr;
            fail("expected ',' or ']'");
        }
    }

    static void append_utf8(std::string& out, uint32_t cp) {
        if (cp < 0x80) {
            out.push_back(static_cast<char>(cp));
        } else if (cp < 0x800) {
            out.push_back(static_cast<char>(0xC0 | (cp >> 6)));
            out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
        } else if (cp < 0x10000) {
            out.push_back(static_cast<char>(0xE0 | (cp >> 12)));
            out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
            out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
        } else {
            out.push_back(static_cast<char>(0xF0 | (cp >> 18)));
            out.push_back(static_cast<char>(0x80 | ((cp >> 12) & 0x3F)));
            out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
            out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
        }
    }
    uint32_t parse_hex4() {
        if (pos_ + 4 > s_.size()) fail("short \\u escape");
        uint32_t v = 0;
        for (int i = 0; i < 4; ++i) {
            const char c = s_[pos_++];
            v <<= 4;
            if (c >= '0' && c <= '9') v |= static_cast<uint32_t>(c - '0');
            else if (c >= 'a' && c <= 'f') v |= static_cast<uint32_t>(c - 'a' + 10);
            else if (c >= 'A' && c <= 'F') v |= static_cast<uint32_t>(c - 'A' + 10);
            else fail("bad \\u escape");
        }
        return v;
    }
    std::string parse_string() {
        std::string out;
        ++pos_;  // opening quote
        for (;;) {
            if (pos_ >= s_.size()) fail("unterminated string");
            const unsigned char c = static_cast<unsigned char>(s_[pos_++]);
            if (c == '"') return out;
            if (c < 0x20) fail("control character in string");
            if (c != '\\') {
                out.push_back(static_cast<char>(c));
                continue;
            }
            if (pos_ >= s_.size()) fail("unterminated escape");
            const char e = s_[pos_++];
            switch (e) {
                case '"': out.push_back('"'); break;
                case '\\': out.push_back('\\'); break;
                case '/': out.push_back('/'); break;
                case 'b': out.push_back('\b'); break;
                case 'f': out.push_back('\f'); break;
                case 'n': out.push_back('\n'); break;
                case 'r': out.push_back('\r'); break;
                case 't': out.push_back('\t'); break;
                case 'u': {
                    uint32_t cp = parse_hex4();
                    if (cp >= 0xD800 && cp <= 0xDBFF) {  // surrogate pair
                        if (pos_ + 2 > s_.size() || s_[pos_] != '\\' || s_[pos_ + 1] != 'u') fail("lone surrogate");
                        pos_ += 2;
                        const uint32_t lo = parse_hex4();
                        if (lo < 0xDC00 || lo > 0xDFFF) fail("bad surrogate pair");
                        cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                    } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
                        fail("lone surrogate");
                    }
                    append_utf8(out, cp);
                    break;
                }
                default: fail("bad escape");
            }
        }
    }

    Value parse_number() {
        const size_t start = pos_;
        bool is_real = false;
        if (eat('-')) {}
        if (pos_ >= s_.size()) fail("bad number");
        if (s_[pos_] == '0') {
            ++pos_;
        } else if (s_[pos_] >= '1' && s_[pos_] <= '9') {
            while (pos_ < s_.size() && s_[pos_] >= '0' && s_[pos_] <= '9') ++pos_;
        } else {
            fail("bad number");
        }
        if (pos_ < s_.size() && s_[pos_] == '.') {
            is_real = true;
            ++pos_;
            if (pos_ >= s_.size() || s_[pos_] < '0' || s_[pos_] > '9') fail("bad fraction");
            while (pos_ < s_.size() && s_[pos_] >= '0' && s_[pos_] <= '9') ++pos_;
        }
        if (pos_ < s_.size() && (s_[pos_] == 'e' || s_[pos_] == 'E')) {
            is_real = true;
            ++pos_;
            if (pos_ < s_.size() && (s_[pos_] == '+' || s_[pos_] == '-')) ++pos_;
            if (pos_ >= s_.size() || s_[pos_] < '0' || s_[pos_] > '9') fail("bad exponent");
            while (pos_ < s_.size() && s_[pos_] >= '0' && s_[pos_] <= '9') ++pos_;
        }
        const char* b = s_.data() + start;
        const char* e = s_.data() + pos_;
        if (!is_real) {
            int64_t iv = 0;
            auto r = std::from_chars(b, e, iv);
            if (r.ec == std::errc() && r.ptr == e) return Value::integer(iv);
            // does not fit in 64 bits: keep it as a real, like any other out-of-range literal
        }
        double dv = 0.0;
        auto r = std::from_chars(b, e, dv);
        if (r.ec == std::errc::result_out_of_range) fail("number out of range");
        if (r.ec != std::errc() || r.ptr != e) fail("bad number");
        return Value::real(dv);
    }
};

inline Value parse(std::string_view text) { return Parser(text).parse_document(); }

// ---------------------------------------------------------------------------------------------
// printer
// ---------------------------------------------------------------------------------------------
// Shortest digits that round-trip, laid out as: plain integer part + ".0" when the value is
// integral and below 1e15, positional notation for decimal exponents in (-4, 15], scientific with
// a sign and at least two exponent digits otherwise.  Non-finite values print as null.
inline void append_real(std::string& out, double v) {
    if (!std::isfinite(v)) {
        out += "null";
        return;
    }
    if (std::signbit(v)) {
        out.push_back('-');
        v = -v;
    }
    if (v == 0.0) {
        out += "0.0";
        return;
    }
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::scientific);
    std::string_view sci(buf, static_cast<size_t>(r.ptr - buf));  // d[.ddd]e[+-]XX
    const size_t epos = sci.find('e');
    std::string digits;
    for (char c : sci.substr(0, epos))
        if (c != '.') digits.push_back(c);
    int exp10 = 0;
    std::from_chars(sci.data() + epos + 1 + (sci[epos + 1] == '+' ? 1 : 0), sci.data() + sci.size(), exp10);
    const int k = static_cast<int>(digits.size());
    const int n = exp10 + 1;  // position of the decimal point relative to the first digit
    constexpr int kMinExp = -4, kMaxExp = 15;
    if (k <= n && n <= kMaxExp) {
        out += digits;
        out.append(static_cast<size_t>(n - k), '0');
        out += ".0";
    } else if (0 < n && n <= kMaxExp) {
        out.append(digits, 0, static_cast<size_t>(n));
        out.push_back('.');
        out.append(digits, static_cast<size_t>(n), std::string::npos);
    } else if (kMinExp < n && n <= 0) {
        out += "0.";
        out.append(static_cast<size_t>(-n), '0');
        out += digits;
    } else {
        out.push_back(digits[0]);
        if (k > 1) {
            out.push_back('.');
            out.append(digits, 1, std::string::npos);
        }
        out.push_back('e');
        int e = n - 1;
        out.push_back(e < 0 ? '-' : '+');
        if (e < 0) e = -e;
        if (e < 10) out.push_back('0');
        out += std::to_string(e);
    }
}

inline void append_string(std::string& out, std::string_view s) {
    out.push_back('"');
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
                    char tmp[8];
                    std::snprintf(tmp, sizeof(tmp), "\\u%04x", c);
                    out += tmp;
                } else {
                    out.push_back(static_cast<char>(c));
                }
        }
    }
    out.push_back('"');
}

inline void dump(const Value& v, std::string& out, int indent, int level = 0) {
    switch (v.kind()) {
        case Value::Kind::Null: out += "null"; break;
        case Value::Kind::Bool: out += v.as_int() ? "true" : "false"; break;
        case Value::Kind::Int: out += std::to_string(v.as_int()); break;
        case Value::Kind::Real: append_real(out, v.as_real()); break;
        case Value::Kind::String: append_string(out, v.as_string()); break;
        case Value::Kind::Array: {
            if (v.items().empty()) {
                out += "[]";
                break;
            }
            out += "[\n";
            for (size_t i = 0; i < v.items().size(); ++i) {
                out.append(static_cast<size_t>((level + 1) * indent), ' ');
                dump(v.items()[i], out, indent, level + 1);
                out += i + 1 < v.items().size() ? ",\n" : "\n";
            }
            out.append(static_cast<size_t>(level * indent), ' ');
            out.push_back(']');
            break;
        }
        case Value::Kind::Object: {
            if (v.members().empty()) {
                out += "{}";
                break;
            }
            out += "{\n";
            for (size_t i = 0; i < v.members().size(); ++i) {
                out.append(static_cast<size_t>((level + 1) * indent), ' ');
                append_string(out, v.members()[i].first);
                out += ": ";
                dump(v.members()[i].second, out, indent, level + 1);
                out += i + 1 < v.members().size() ? ",\n" : "\n";
            }
            out.append(static_cast<size_t>(level * indent), ' ');
            out.push_back('}');
            break;
        }
    }
}

}  // namespace rfjson
