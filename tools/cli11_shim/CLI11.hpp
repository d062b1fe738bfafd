// CLI11.hpp -- a minimal, independent implementation of the CLI11 subset the
// reference CLI (/root/reference/proj/tools/main.cpp:184-220) uses:
// App::add_option for strings, unsigned integers and delimited vectors,
// Option::required / check / delimiter, IsMember, App::parse, App::exit and
// the ParseError family.  The real CLI11 is vendored by the reference
// (proj/.gitignore:2) and absent from this image; this shim lets the
// reference's unmodified main.cpp be compiled and linked against the B200
// engine.  It is not a copy of CLI11.
#pragma once

#include <cstdint>
#include <cstdio>
#include <functional>
#include <initializer_list>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

class ParseError : public std::runtime_error {
public:
    ParseError(std::string name, const std::string& msg, int code)
        : std::runtime_error(msg), name_(std::move(name)), code_(code) {}
    int get_exit_code() const { return code_; }
    const std::string& get_name() const { return name_; }

private:
    std::string name_;
    int code_;
};

struct CallForHelp : ParseError {
    CallForHelp() : ParseError("CallForHelp", "This should be caught in your main function, see examples", 0) {}
};
struct RequiredError : ParseError {
    explicit RequiredError(const std::string& opt) : ParseError("RequiredError", opt + " is required", 106) {}
};
struct ValidationError : ParseError {
    explicit ValidationError(const std::string& msg) : ParseError("ValidationError", msg, 105) {}
};
struct ConversionError : ParseError {
    explicit ConversionError(const std::string& msg) : ParseError("ConversionError", msg, 103) {}
};
struct ExtrasError : ParseError {
    explicit ExtrasError(const std::string& msg) : ParseError("ExtrasError", msg, 109) {}
};

// A validator returns an empty string when the value is acceptable.
struct Validator {
    std::function<std::string(const std::string&)> fn;
};

inline Validator IsMember(std::initializer_list<const char*> items) {
    std::vector<std::string> set(items.begin(), items.end());
    return Validator{[set](const std::string& v) -> std::string {
        for (const auto& s : set)
            if (s == v) return {};
        std::string all;
        for (const auto& s : set) all += (all.empty() ? "" : ",") + s;
        return v + " not in {" + all + "}";
    }};
}

class Option {
public:
    Option(std::string name, std::function<void(const std::string&)> assign, bool is_vector)
        : name_(std::move(name)), assign_(std::move(assign)), is_vector_(is_vector) {}
    Option* required(bool r = true) {
        required_ = r;
        return this;
    }
    Option* check(Validator v) {
        checks_.push_back(std::move(v));
        return this;
    }
    Option* delimiter(char c) {
        delim_ = c;
        return this;
    }

private:
    friend class App;
    std::string name_;
    std::function<void(const std::string&)> assign_;
    bool is_vector_;
    bool required_ = false;
    bool seen_ = false;
    char delim_ = 0;
    std::vector<Validator> checks_;
};

namespace detail {
template <typename T>
T to_unsigned(const std::string& name, const std::string& s) {
    if (s.empty() || s[0] == '-' || s[0] == '+')
        throw ConversionError("Could not convert: " + name + " = " + s);
    std::size_t pos = 0;
    unsigned long long v = 0;
    try {
        v = std::stoull(s, &pos, 10);
    } catch (...) {
        throw ConversionError("Could not convert: " + name + " = " + s);
    }
    if (pos != s.size() || v > static_cast<unsigned long long>(std::numeric_limits<T>::max()))
        throw ConversionError("Could not convert: " + name + " = " + s);
    return static_cast<T>(v);
}
}  // namespace detail

class App {
public:
    explicit App(std::string description = {}) : description_(std::move(description)) {}

    Option* add_option(const std::string& name, std::string& var, const std::string& = {}) {
        return add(name, [&var](const std::string& s) { var = s; }, false);
    }

    template <typename T, typename = std::enable_if_t<std::is_integral_v<T> && std::is_unsigned_v<T>>>
    Option* add_option(const std::string& name, T& var, const std::string& = {}) {
        return add(name, [&var, name](const std::string& s) { var = detail::to_unsigned<T>(name, s); }, false);
    }

    template <typename T>
    Option* add_option(const std::string& name, std::vector<T>& var, const std::string& = {}) {
        return add(name, [&var, name](const std::string& s) { var.push_back(detail::to_unsigned<T>(name, s)); },
                   true);
    }

    void parse(int argc, char** argv) {
        for (int i = 1; i < argc; ++i) {
            std::string arg = argv[i];
            if (arg == "-h" || arg == "--help") throw CallForHelp();
            std::string value;
            bool has_value = false;
            const auto eq = arg.find('=');
            if (arg.rfind("--", 0) == 0 && eq != std::string::npos) {
                value = arg.substr(eq + 1);
                arg = arg.substr(0, eq);
                has_value = true;
            }
            Option* opt = find(arg);
            if (!opt) throw ExtrasError("The following arguments were not expected: " + std::string(argv[i]));
            if (!has_value) {
                if (i + 1 >= argc) throw ConversionError(arg + " requires an argument");
                value = argv[++i];
            }
            std::vector<std::string> parts;
            if (opt->is_vector_ && opt->delim_) {
                std::string cur;
                for (char c : value) {
                    if (c == opt->delim_) {
                        parts.push_back(cur);
                        cur.clear();
                    } else {
                        cur += c;
                    }
                }
                parts.push_back(cur);
            } else {
                parts.push_back(value);
            }
            for (const auto& part : parts) {
                for (const auto& v : opt->checks_) {
                    const std::string err = v.fn(part);
                    if (!err.empty()) throw ValidationError(arg + ": " + err);
                }
                opt->assign_(part);
            }
            opt->seen_ = true;
        }
        for (const auto& o : options_)
            if (o->required_ && !o->seen_) throw RequiredError(o->name_);
    }

    int exit(const ParseError& e) const {
        if (e.get_exit_code() == 0) {
            std::printf("%s\n", description_.c_str());
            for (const auto& o : options_) std::printf("  %s\n", o->name_.c_str());
            return 0;
        }
        std::fprintf(stderr, "%s\nRun with --help for more information.\n", e.what());
        return e.get_exit_code();
    }

private:
    Option* add(const std::string& name, std::function<void(const std::string&)> assign, bool is_vector) {
        options_.push_back(std::make_unique<Option>(name, std::move(assign), is_vector));
        return options_.back().get();
    }
    Option* find(const std::string& name) {
        for (auto& o : options_)
            if (o->name_ == name) return o.get();
        return nullptr;
    }

    std::string description_;
    std::vector<std::unique_ptr<Option>> options_;
};

}  // namespace CLI
