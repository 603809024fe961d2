// CLI11.hpp — a minimal stand-in for the CLI11 command-line library, enough
// to compile the reference's tools/main.cpp (the `sirdfit` CLI).
//
// TEST INFRASTRUCTURE.  The reference vendors CLI11 under proj/vendor/, which
// is git-ignored and not shipped (SURVEY.md §0 finding 5), so its CLI cannot
// be built as delivered.  This header implements only the surface main.cpp
// uses — App with subcommands, typed options and flags, required options,
// the ExistingFile / PositiveNumber / IsMember validators, a `--config` file
// of `key = value` lines, CLI11_PARSE — so oracle/Makefile can build the
// reference's unmodified CLI against the pure reference and against the B200
// binding (ref_binding/) and compare their outputs byte for byte.
#pragma once

#include <charconv>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <functional>
#include <initializer_list>
#include <iostream>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

struct Error : std::runtime_error {
    int code;
    Error(const std::string& msg, int c) : std::runtime_error(msg), code(c) {}
};
struct ParseError : Error {
    explicit ParseError(const std::string& m) : Error(m, 109) {}
};
struct ValidationError : Error {
    explicit ValidationError(const std::string& m) : Error(m, 105) {}
};
struct RequiredError : Error {
    explicit RequiredError(const std::string& m) : Error(m, 106) {}
};
struct CallForHelp : Error {
    CallForHelp() : Error("help", 0) {}
};

// A validator returns an empty string for a valid value, else the message.
using Validator = std::function<std::string(const std::string&)>;

inline const Validator ExistingFile = [](const std::string& s) -> std::string {
    return std::filesystem::is_regular_file(s) ? "" : "File does not exist: " + s;
};

inline const Validator PositiveNumber = [](const std::string& s) -> std::string {
    char* end = nullptr;
    const double v = std::strtod(s.c_str(), &end);
    return end && *end == '\0' && v > 0.0 ? "" : "Value " + s + " not a positive number";
};

inline Validator IsMember(std::initializer_list<const char*> allowed) {
    std::vector<std::string> set(allowed.begin(), allowed.end());
    return [set](const std::string& s) -> std::string {
        for (const std::string& a : set)
            if (a == s) return "";
        return s + " not in the allowed set";
    };
}

namespace detail {

template <class T>
void convert(const std::string& s, T& out) {
    if constexpr (std::is_same_v<T, std::string>) {
        out = s;
    } else if constexpr (std::is_floating_point_v<T>) {
        char* end = nullptr;
        const double v = std::strtod(s.c_str(), &end);
        if (s.empty() || !end || *end != '\0') throw ParseError("could not convert " + s + " to a number");
        out = static_cast<T>(v);
    } else {
        static_assert(std::is_integral_v<T>, "unsupported option type");
        T v{};
        const auto r = std::from_chars(s.data(), s.data() + s.size(), v);
        if (s.empty() || r.ec != std::errc() || r.ptr != s.data() + s.size())
            throw ParseError("could not convert " + s + " to an integer");
        out = v;
    }
}

}  // namespace detail

class Option {
public:
    Option(std::string name, std::function<void(const std::string&)> set, bool flag)
        : name_(std::move(name)), set_(std::move(set)), flag_(flag) {}
    Option* required(bool value = true) {
        required_ = value;
        return this;
    }
    Option* check(Validator v) {
        checks_.push_back(std::move(v));
        return this;
    }
    Option* capture_default_str() { return this; }

    const std::string& name() const { return name_; }
    bool flag() const { return flag_; }
    bool is_required() const { return required_; }
    std::size_t count() const { return count_; }

    void apply(const std::string& value) {
        for (const Validator& v : checks_) {
            const std::string msg = v(value);
            if (!msg.empty()) throw ValidationError(name_ + ": " + msg);
        }
        set_(value);
        ++count_;
    }

private:
    std::string name_;
    std::function<void(const std::string&)> set_;
    bool flag_;
    bool required_ = false;
    std::size_t count_ = 0;
    std::vector<Validator> checks_;
};

class App {
public:
    explicit App(std::string description = "", std::string name = "")
        : description_(std::move(description)), name_(std::move(name)) {}

    void set_config(std::string option_name) { config_option_ = std::move(option_name); }
    void require_subcommand(int n) { require_subcommands_ = n; }

    App* add_subcommand(std::string name, std::string description = "") {
        subcommands_.push_back(std::make_unique<App>(std::move(description), std::move(name)));
        return subcommands_.back().get();
    }

    template <class T>
    Option* add_option(std::string name, T& target, std::string /*description*/ = "") {
        options_.push_back(std::make_unique<Option>(
            std::move(name), [&target](const std::string& s) { detail::convert(s, target); }, false));
        return options_.back().get();
    }

    Option* add_flag(std::string name, bool& target, std::string /*description*/ = "") {
        options_.push_back(std::make_unique<Option>(
            std::move(name), [&target](const std::string&) { target = true; }, true));
        return options_.back().get();
    }

    bool parsed() const { return parsed_; }

    void parse(int argc, char** argv) {
        std::vector<std::string> args(argv + 1, argv + argc);
        std::size_t k = 0;
        App* target = this;
        std::string config_file;
        while (k < args.size()) {
            const std::string& a = args[k];
            if (a == "-h" || a == "--help") throw CallForHelp();
            if (target == this && a.rfind("-", 0) != 0) {
                App* sub = find_subcommand(a);
                if (!sub) throw ParseError("unknown subcommand " + a);
                sub->parsed_ = true;
                target = sub;
                ++k;
                continue;
            }
            std::string name = a, value;
            bool inline_value = false;
            if (const auto eq = a.find('='); a.rfind("--", 0) == 0 && eq != std::string::npos) {
                name = a.substr(0, eq);
                value = a.substr(eq + 1);
                inline_value = true;
            }
            if (!config_option_.empty() && name == config_option_) {
                if (!inline_value) {
                    if (k + 1 >= args.size()) throw ParseError(name + " needs a value");
                    value = args[++k];
                }
                config_file = value;
                ++k;
                continue;
            }
            Option* opt = target->find_option(name);
            if (!opt) throw ParseError("the following argument was not expected: " + a);
            if (opt->flag()) {
                opt->apply("true");
            } else {
                if (!inline_value) {
                    if (k + 1 >= args.size()) throw ParseError(name + " needs a value");
                    value = args[++k];
                }
                opt->apply(value);
            }
            ++k;
        }
        if (require_subcommands_ > 0 && target == this) throw RequiredError("A subcommand is required");
        parsed_ = true;
        if (!config_file.empty()) target->apply_config(config_file);
        target->check_required();
    }

    int exit(const Error& e) const {
        if (dynamic_cast<const CallForHelp*>(&e)) {
            std::cout << description_ << "\n";
            return 0;
        }
        std::cerr << e.what() << "\n";
        return e.code;
    }

private:
    App* find_subcommand(const std::string& name) {
        for (auto& s : subcommands_)
            if (s->name_ == name) return s.get();
        return nullptr;
    }
    Option* find_option(const std::string& name) {
        for (auto& o : options_)
            if (o->name() == name) return o.get();
        return nullptr;
    }
    // `key = value` lines (options given on the command line take precedence)
    void apply_config(const std::string& path) {
        std::ifstream in(path);
        if (!in) throw ParseError("cannot read config file " + path);
        std::string line;
        while (std::getline(in, line)) {
            const auto hash = line.find('#');
            if (hash != std::string::npos) line.resize(hash);
            const auto eq = line.find('=');
            if (eq == std::string::npos) continue;
            auto trim = [](std::string s) {
                const auto b = s.find_first_not_of(" \t\"");
                const auto e = s.find_last_not_of(" \t\"\r");
                return b == std::string::npos ? std::string() : s.substr(b, e - b + 1);
            };
            const std::string key = "--" + trim(line.substr(0, eq)), value = trim(line.substr(eq + 1));
            Option* opt = find_option(key);
            if (!opt) throw ParseError("unknown config key " + key);
            if (opt->count() == 0) opt->apply(opt->flag() ? "true" : value);
        }
    }
    void check_required() const {
        for (const auto& o : options_)
            if (o->is_required() && o->count() == 0) throw RequiredError(o->name() + " is required");
    }

    std::string description_, name_, config_option_;
    int require_subcommands_ = 0;
    bool parsed_ = false;
    std::vector<std::unique_ptr<App>> subcommands_;
    std::vector<std::unique_ptr<Option>> options_;
};

}  // namespace CLI

#define CLI11_PARSE(app, argc, argv)              \
    try {                                         \
        (app).parse((argc), (argv));              \
    } catch (const CLI::Error& cli_error_) {      \
        return (app).exit(cli_error_);            \
    }
