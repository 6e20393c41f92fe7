// Minimal JSON for the trace contract (the reference uses nlohmann/json,
// which is not vendored here): flat objects with sorted keys, doubles as that
// library prints them (grisu2.hpp), and a small parser for Trace::from_jsonl.
#pragma once

#include <charconv>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "grisu2.hpp"

namespace asyrk::json {

struct Value;
using Object = std::map<std::string, Value>;
using Array = std::vector<Value>;

struct Value {
    std::variant<std::nullptr_t, bool, int64_t, double, std::string, std::shared_ptr<Array>, std::shared_ptr<Object>> v;
    Value() : v(nullptr) {}
    Value(bool b) : v(b) {}
    Value(int x) : v(static_cast<int64_t>(x)) {}
    Value(int64_t x) : v(x) {}
    Value(uint64_t x) : v(static_cast<int64_t>(x)) {}
    Value(double x) : v(x) {}
    Value(const char* s) : v(std::string(s)) {}
    Value(std::string s) : v(std::move(s)) {}
    Value(Array a) : v(std::make_shared<Array>(std::move(a))) {}
    Value(Object o) : v(std::make_shared<Object>(std::move(o))) {}

    bool is_object() const { return std::holds_alternative<std::shared_ptr<Object>>(v); }
    bool is_array() const { return std::holds_alternative<std::shared_ptr<Array>>(v); }
    const Object& object() const { return *std::get<std::shared_ptr<Object>>(v); }
    const Array& array() const { return *std::get<std::shared_ptr<Array>>(v); }
    double number() const {
        if (auto p = std::get_if<double>(&v)) return *p;
        if (auto p = std::get_if<int64_t>(&v)) return static_cast<double>(*p);
        throw std::runtime_error("json: not a number");
    }
    int64_t integer() const {
        if (auto p = std::get_if<int64_t>(&v)) return *p;
        if (auto p = std::get_if<double>(&v)) return static_cast<int64_t>(*p);
        throw std::runtime_error("json: not an integer");
    }
};

inline void dump_string(const std::string& s, std::string& out) {
    out += '"';
    for (char c : s) {
        switch (c) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\n': out += "\\n"; break;
            case '\t': out += "\\t"; break;
            default: out += c;
        }
    }
    out += '"';
}

inline void dump_double(double d, std::string& out) {
    if (d != d || d == 1.0 / 0.0 || d == -1.0 / 0.0) {
        out += "null";  // nlohmann's convention for non-finite
        return;
    }
    grisu2::to_string(d, out);  // the reference serializer's digits and layout
}

inline void dump(const Value& v, std::string& out) {
    struct V {
        std::string& o;
        void operator()(std::nullptr_t) { o += "null"; }
        void operator()(bool b) { o += b ? "true" : "false"; }
        void operator()(int64_t x) { o += std::to_string(x); }
        void operator()(double d) { dump_double(d, o); }
        void operator()(const std::string& s) { dump_string(s, o); }
        void operator()(const std::shared_ptr<Array>& a) {
            o += '[';
            for (std::size_t k = 0; k < a->size(); ++k) {
                if (k) o += ',';
                dump((*a)[k], o);
            }
            o += ']';
        }
        void operator()(const std::shared_ptr<Object>& ob) {
            o += '{';
            bool first = true;
            for (const auto& [k, val] : *ob) {
                if (!first) o += ',';
                first = false;
                dump_string(k, o);
                o += ':';
                dump(val, o);
            }
            o += '}';
        }
    };
    std::visit(V{out}, v.v);
}

inline std::string dump(const Value& v) {
    std::string s;
    dump(v, s);
    return s;
}

class Parser {
  public:
    explicit Parser(const std::string& t) : t_(t) {}
    Value parse() {
        Value v = value();
        ws();
        if (p_ != t_.size()) throw std::runtime_error("json: trailing characters");
        return v;
    }

  private:
    const std::string& t_;
    std::size_t p_ = 0;
    void ws() {
        while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\n' || t_[p_] == '\r' || t_[p_] == '\t')) ++p_;
    }
    char peek() {
        ws();
        if (p_ >= t_.size()) throw std::runtime_error("json: unexpected end");
        return t_[p_];
    }
    void expect(char c) {
        if (peek() != c) throw std::runtime_error(std::string("json: expected ") + c);
        ++p_;
    }
    Value value() {
        const char c = peek();
        if (c == '{') return object();
        if (c == '[') return array();
        if (c == '"') return Value(str());
        if (t_.compare(p_, 4, "true") == 0) return p_ += 4, Value(true);
        if (t_.compare(p_, 5, "false") == 0) return p_ += 5, Value(false);
        if (t_.compare(p_, 4, "null") == 0) return p_ += 4, Value();
        return number();
    }
    std::string str() {
        expect('"');
        std::string s;
        while (p_ < t_.size() && t_[p_] != '"') {
            if (t_[p_] == '\\' && p_ + 1 < t_.size()) {
                const char e = t_[++p_];
                s += e == 'n' ? '\n' : e == 't' ? '\t' : e;
            } else {
                s += t_[p_];
            }
            ++p_;
        }
        expect('"');
        return s;
    }
    Value number() {
        const std::size_t b = p_;
        bool is_float = false;
        while (p_ < t_.size() && std::string("+-0123456789.eE").find(t_[p_]) != std::string::npos) {
            if (t_[p_] == '.' || t_[p_] == 'e' || t_[p_] == 'E') is_float = true;
            ++p_;
        }
        if (b == p_) throw std::runtime_error("json: bad value");
        if (!is_float) {
            int64_t x = 0;
            auto r = std::from_chars(t_.data() + b, t_.data() + p_, x);
            if (r.ec == std::errc()) return Value(x);
        }
        double d = 0.0;
        auto r = std::from_chars(t_.data() + b, t_.data() + p_, d);
        if (r.ec != std::errc()) throw std::runtime_error("json: bad number");
        return Value(d);
    }
    Value array() {
        expect('[');
        Array a;
        if (peek() == ']') return ++p_, Value(std::move(a));
        for (;;) {
            a.push_back(value());
            if (peek() == ',') {
                ++p_;
                continue;
            }
            expect(']');
            return Value(std::move(a));
        }
    }
    Value object() {
        expect('{');
        Object o;
        if (peek() == '}') return ++p_, Value(std::move(o));
        for (;;) {
            std::string k = str();
            expect(':');
            o[k] = value();
            if (peek() == ',') {
                ++p_;
                continue;
            }
            expect('}');
            return Value(std::move(o));
        }
    }
};

inline Value parse(const std::string& t) { return Parser(t).parse(); }

}  // namespace asyrk::json
