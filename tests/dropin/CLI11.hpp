// TEST INFRASTRUCTURE ONLY -- a minimal stand-in for the CLI11 header the
// reference's tools/cbench.cpp includes (CLI11 is not in this image). It
// implements the subset cbench uses -- App with subcommands, add_option /
// add_flag bound to variables, default_val, required, take_all, expected,
// check(IsMember), require_subcommand, parse, exit, parsed, ParseError -- so
// the UNMODIFIED cbench.cpp compiles against the B200 drop-in headers
// (tests/dropin/Makefile) and against the reference (for comparison).
#pragma once

#include <cstdint>
#include <functional>
#include <iostream>
#include <memory>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace CLI {

class ParseError : public std::runtime_error {
public:
    ParseError(const std::string& m, int code) : std::runtime_error(m), code_(code) {}
    int get_exit_code() const { return code_; }

private:
    int code_;
};

struct IsMember {
    std::set<std::string> allowed;
    IsMember(std::initializer_list<const char*> l) {
        for (const char* s : l) allowed.insert(s);
    }
};

class Option {
public:
    std::string name;
    bool is_flag = false, required_ = false, vector = false, seen = false;
    int expected_ = 1;  // values per occurrence (vector + take_all: -1)
    std::set<std::string> member;
    std::function<void(const std::string&)> assign;
    std::function<void()> clear;

    Option* required() {
        required_ = true;
        return this;
    }
    Option* take_all() {
        expected_ = -1;
        return this;
    }
    Option* expected(int n) {
        expected_ = n;
        return this;
    }
    Option* check(const IsMember& m) {
        member = m.allowed;
        return this;
    }
    template <class T>
    Option* default_val(const T& v) {
        std::ostringstream ss;
        ss << v;
        assign(ss.str());
        return this;
    }
};

namespace detail {
template <class T>
void parse_value(const std::string& s, T& out) {
    std::istringstream ss(s);
    ss >> out;
    if (ss.fail() || !ss.eof()) throw ParseError("invalid value \"" + s + "\"", 1);
}
inline void parse_value(const std::string& s, std::string& out) { out = s; }
}  // namespace detail

class App {
public:
    explicit App(std::string description = "", std::string name = "") : desc_(std::move(description)), name_(std::move(name)) {}

    App* add_subcommand(const std::string& name, const std::string& description = "") {
        subs_.push_back(std::make_unique<App>(description, name));
        return subs_.back().get();
    }
    void require_subcommand(int n) { need_sub_ = n; }

    template <class T>
    Option* add_option(const std::string& name, T& var, const std::string& = "") {
        auto o = std::make_unique<Option>();
        o->name = name;
        o->assign = [&var](const std::string& s) { detail::parse_value(s, var); };
        opts_.push_back(std::move(o));
        return opts_.back().get();
    }
    template <class T>
    Option* add_option(const std::string& name, std::vector<T>& var, const std::string& = "") {
        auto o = std::make_unique<Option>();
        o->name = name;
        o->vector = true;
        o->expected_ = -1;
        o->assign = [&var](const std::string& s) {
            T v{};
            detail::parse_value(s, v);
            var.push_back(v);
        };
        o->clear = [&var] { var.clear(); };
        opts_.push_back(std::move(o));
        return opts_.back().get();
    }
    Option* add_flag(const std::string& name, bool& var, const std::string& = "") {
        auto o = std::make_unique<Option>();
        o->name = name;
        o->is_flag = true;
        o->assign = [&var](const std::string&) { var = true; };
        opts_.push_back(std::move(o));
        return opts_.back().get();
    }

    bool parsed() const { return parsed_; }

    void parse(int argc, char** argv) {
        std::vector<std::string> args(argv + 1, argv + argc);
        parse_args(args, 0);
    }

    int exit(const ParseError& e) const {
        if (e.get_exit_code() == 0) {
            std::cout << help();
        } else {
            std::cerr << e.what() << "\n" << "Run with --help for more information.\n";
        }
        return e.get_exit_code();
    }

private:
    std::string help() const {
        std::string h = (name_.empty() ? std::string("cbench") : name_) + ": " + desc_ + "\n";
        for (const auto& s : subs_) h += "  " + s->name_ + "  " + s->desc_ + "\n";
        for (const auto& o : opts_) h += "  " + o->name + "\n";
        return h;
    }
    Option* find(const std::string& n) {
        for (auto& o : opts_)
            if (o->name == n) return o.get();
        return nullptr;
    }
    void parse_args(const std::vector<std::string>& a, size_t i) {
        parsed_ = true;
        while (i < a.size()) {
            const std::string& t = a[i];
            if (t == "--help" || t == "-h") throw ParseError("help", 0);
            if (t.rfind("--", 0) == 0) {
                std::string key = t, inline_val;
                const bool has_eq = t.find('=') != std::string::npos;
                if (has_eq) {
                    key = t.substr(0, t.find('='));
                    inline_val = t.substr(t.find('=') + 1);
                }
                Option* o = find(key);
                if (!o) throw ParseError("The following argument was not expected: " + t, 1);
                ++i;
                if (o->is_flag) {
                    o->assign("");
                    o->seen = true;
                    continue;
                }
                if (o->vector && !o->seen && o->clear) o->clear();
                std::vector<std::string> vals;
                if (has_eq) vals.push_back(inline_val);
                const int want = o->expected_;
                while (i < a.size() && (want < 0 || (int)vals.size() < want) && a[i].rfind("--", 0) != 0) vals.push_back(a[i++]);
                if (vals.empty() || (want > 0 && (int)vals.size() != want))
                    throw ParseError(key + ": expected " + (want > 0 ? std::to_string(want) : std::string("at least 1")) +
                                         " argument(s)",
                                     1);
                for (const auto& v : vals) {
                    if (!o->member.empty() && !o->member.count(v))
                        throw ParseError(key + ": " + v + " not in the allowed set", 1);
                    o->assign(v);
                }
                o->seen = true;
                continue;
            }
            App* sub = nullptr;
            for (auto& s : subs_)
                if (s->name_ == t) sub = s.get();
            if (!sub) throw ParseError("The following argument was not expected: " + t, 1);
            sub->parse_args(a, i + 1);
            i = a.size();
            ++nsub_;
        }
        for (auto& o : opts_)
            if (o->required_ && !o->seen) throw ParseError(o->name + " is required", 1);
        if (need_sub_ > 0 && nsub_ < need_sub_) throw ParseError("A subcommand is required", 1);
    }

    std::string desc_, name_;
    std::vector<std::unique_ptr<App>> subs_;
    std::vector<std::unique_ptr<Option>> opts_;
    int need_sub_ = 0, nsub_ = 0;
    bool parsed_ = false;
};

}  // namespace CLI
