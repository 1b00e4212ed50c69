// Minimal stand-in for the CLI11 header the reference's tools/pint_bench.cpp includes (CLI11 is
// not vendored in the reference, proj/.gitignore). Just the surface pint_bench uses: an App with
// subcommands and typed options (scalars, strings, comma-delimited vectors), IsMember / Range
// checks, capture_default_str (a no-op), ParseError + App::exit. Test/build infrastructure only
// (oracle/Makefile target `dropin` builds the reference's pint_bench against the B200 drop-in).
#pragma once

#include <functional>
#include <iostream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

struct ParseError : std::runtime_error {
    int code;
    ParseError(const std::string& what, int c) : std::runtime_error(what), code(c) {}
};

using Validator = std::function<std::string(const std::string&)>;  // "" = ok, else the error

inline Validator IsMember(std::vector<std::string> allowed) {
    return [allowed](const std::string& v) {
        for (const auto& a : allowed)
            if (a == v) return std::string();
        return "value " + v + " not in the allowed set";
    };
}

inline Validator Range(double lo, double hi) {
    return [lo, hi](const std::string& v) {
        const double x = std::stod(v);
        return (x < lo || x > hi) ? "value " + v + " out of range" : std::string();
    };
}

namespace detail {
template <class T>
void assign(T& out, const std::string& s) {
    std::istringstream in(s);
    in >> out;
    if (in.fail()) throw ParseError("cannot parse '" + s + "'", 2);
}
inline void assign(std::string& out, const std::string& s) { out = s; }
}  // namespace detail

class Option {
  public:
    template <class T>
    Option(std::string name, T& var) : name_(std::move(name)) {
        set_ = [&var, this](const std::string& s) {
            if constexpr (std::is_same_v<T, std::vector<double>> || std::is_same_v<T, std::vector<std::size_t>> ||
                          std::is_same_v<T, std::vector<int>>) {
                var.clear();
                std::string item;
                std::istringstream in(s);
                while (std::getline(in, item, delim_ ? delim_ : '\n')) {
                    typename T::value_type x{};
                    detail::assign(x, item);
                    var.push_back(x);
                }
            } else {
                detail::assign(var, s);
            }
        };
    }
    Option* check(Validator v) {
        checks_.push_back(std::move(v));
        return this;
    }
    Option* capture_default_str() { return this; }
    Option* delimiter(char d) {
        delim_ = d;
        return this;
    }
    const std::string& name() const { return name_; }
    void take(const std::string& v) {
        for (const auto& c : checks_)
            if (const std::string err = c(v); !err.empty()) throw ParseError(name_ + ": " + err, 2);
        set_(v);
    }

  private:
    std::string name_;
    std::function<void(const std::string&)> set_;
    std::vector<Validator> checks_;
    char delim_ = 0;
};

class App {
  public:
    explicit App(std::string description = "") : description_(std::move(description)) {}
    void require_subcommand(int) {}
    App* add_subcommand(const std::string& name, const std::string& description) {
        subs_.push_back(std::make_unique<App>(description));
        subs_.back()->name_ = name;
        return subs_.back().get();
    }
    template <class T>
    Option* add_option(const std::string& name, T& var, const std::string& = "") {
        options_.push_back(std::make_unique<Option>(name, var));
        return options_.back().get();
    }
    explicit operator bool() const { return parsed_; }

    void parse(int argc, char** argv) {
        if (argc < 2) throw ParseError(usage(), 106);
        const std::string cmd = argv[1];
        if (cmd == "--help" || cmd == "-h") throw ParseError(usage(), 0);
        for (auto& s : subs_)
            if (s->name_ == cmd) {
                s->parsed_ = true;
                for (int i = 2; i < argc; ++i) {
                    const std::string key = argv[i];
                    Option* o = s->find(key);
                    if (!o) throw ParseError("unknown option " + key, 109);
                    if (i + 1 >= argc) throw ParseError(key + " needs a value", 107);
                    o->take(argv[++i]);
                }
                return;
            }
        throw ParseError("unknown subcommand " + cmd + "\n" + usage(), 109);
    }
    int exit(const ParseError& e) const {
        (e.code == 0 ? std::cout : std::cerr) << e.what() << "\n";
        return e.code;
    }

  private:
    Option* find(const std::string& key) {
        for (auto& o : options_)
            if (o->name() == key) return o.get();
        return nullptr;
    }
    std::string usage() const {
        std::string u = description_ + "\nsubcommands:";
        for (const auto& s : subs_) u += "\n  " + s->name_ + "  " + s->description_;
        return u;
    }
    std::string name_, description_;
    bool parsed_ = false;
    std::vector<std::unique_ptr<App>> subs_;
    std::vector<std::unique_ptr<Option>> options_;
};

}  // namespace CLI
