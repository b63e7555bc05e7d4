// TEST INFRASTRUCTURE ONLY — part of the parity oracle under oracle/.
//
// A minimal CLI11-compatible argument parser covering exactly the surface the
// reference CLI (`/root/reference/proj/tools/lynx_main.cpp:230-270`) uses, so
// that the reference's own `lynx` binary builds unmodified into oracle/_ref/
// (CLI11 is not installed in this image). Supported: App with subcommands,
// positional and `--name value` / `--name=value` options of string/integral
// type, boolean flags, ->required(), ->check(IsMember({...})),
// require_subcommand(n), parsed(), CLI11_PARSE. Parse failures print a
// message and exit with CLI11's codes (105 validation, 106 required,
// 109 extras).
#pragma once

#include <functional>
#include <initializer_list>
#include <iostream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

struct Error : std::runtime_error {
  Error(const std::string& what, int code) : std::runtime_error(what), exit_code(code) {}
  int exit_code;
};
struct ParseError : Error {
  ParseError(const std::string& what, int code) : Error(what, code) {}
};
struct ValidationError : ParseError {
  explicit ValidationError(const std::string& what) : ParseError(what, 105) {}
};
struct RequiredError : ParseError {
  explicit RequiredError(const std::string& what) : ParseError(what, 106) {}
};
struct ExtrasError : ParseError {
  explicit ExtrasError(const std::string& what) : ParseError(what, 109) {}
};
struct CallForHelp : ParseError {
  CallForHelp() : ParseError("help", 0) {}
};

struct Validator {
  std::function<std::string(const std::string&)> fn;
};

inline Validator IsMember(std::initializer_list<std::string> items) {
  std::vector<std::string> v(items);
  return {[v](const std::string& s) -> std::string {
    for (const auto& x : v)
      if (x == s) return {};
    return "value '" + s + "' not in the allowed set";
  }};
}

class Option {
 public:
  Option(std::string name, std::function<void(const std::string&)> set, bool flag)
      : name_(std::move(name)), set_(std::move(set)), flag_(flag) {}
  Option* required(bool r = true) {
    required_ = r;
    return this;
  }
  Option* check(Validator v) {
    checks_.push_back(std::move(v));
    return this;
  }

 private:
  friend class App;
  std::string name_;
  std::function<void(const std::string&)> set_;
  bool flag_;
  bool required_ = false;
  bool seen_ = false;
  std::vector<Validator> checks_;
  bool positional() const { return name_.rfind("-", 0) != 0; }
  void assign(const std::string& v) {
    for (auto& c : checks_) {
      std::string err = c.fn(v);
      if (!err.empty()) throw ValidationError(name_ + ": " + err);
    }
    set_(v);
    seen_ = true;
  }
};

template <class T>
void convert(const std::string& s, T& out) {
  if constexpr (std::is_same_v<T, std::string>) {
    out = s;
  } else if constexpr (std::is_same_v<T, bool>) {
    out = (s == "1" || s == "true");
  } else if constexpr (std::is_integral_v<T>) {
    std::size_t pos = 0;
    long long v = 0;
    try {
      v = std::stoll(s, &pos);
    } catch (...) {
      throw ValidationError("expected an integer, got '" + s + "'");
    }
    if (pos != s.size()) throw ValidationError("expected an integer, got '" + s + "'");
    out = static_cast<T>(v);
  } else {
    std::istringstream is(s);
    is >> out;
  }
}

class App {
 public:
  explicit App(std::string desc = "", std::string name = "") : desc_(std::move(desc)), name_(std::move(name)) {}

  void require_subcommand(int n) { need_sub_ = n; }

  App* add_subcommand(const std::string& name, const std::string& desc) {
    subs_.push_back(std::make_unique<App>(desc, name));
    return subs_.back().get();
  }

  template <class T>
  Option* add_option(const std::string& name, T& var, const std::string& = "") {
    opts_.push_back(std::make_unique<Option>(
        name, [&var](const std::string& s) { convert(s, var); }, false));
    return opts_.back().get();
  }

  Option* add_flag(const std::string& name, bool& var, const std::string& = "") {
    opts_.push_back(std::make_unique<Option>(
        name, [&var](const std::string&) { var = true; }, true));
    return opts_.back().get();
  }

  bool parsed() const { return parsed_; }

  void parse(int argc, const char* const* argv) {
    std::vector<std::string> args;
    for (int i = 1; i < argc; ++i) args.emplace_back(argv[i]);
    parse_args(args, 0);
  }

  int exit(const Error& e) const {
    if (e.exit_code == 0) {
      std::cout << desc_ << "\n";
      return 0;
    }
    std::cerr << e.what() << "\n";
    return e.exit_code;
  }

 private:
  void parse_args(const std::vector<std::string>& args, std::size_t i) {
    parsed_ = true;
    std::size_t positional_idx = 0;
    for (; i < args.size(); ++i) {
      const std::string& a = args[i];
      if (a == "--help" || a == "-h") throw CallForHelp();
      if (a.rfind("-", 0) == 0) {
        std::string key = a, val;
        bool has_eq = false;
        auto eq = a.find('=');
        if (eq != std::string::npos) {
          key = a.substr(0, eq);
          val = a.substr(eq + 1);
          has_eq = true;
        }
        Option* o = find(key);
        if (!o) throw ExtrasError("unknown option " + key);
        if (o->flag_) {
          o->assign("1");
        } else {
          if (!has_eq) {
            if (i + 1 >= args.size()) throw ParseError(key + " needs a value", 114);
            val = args[++i];
          }
          o->assign(val);
        }
        continue;
      }
      if (App* s = find_sub(a)) {
        s->parse_args(args, i + 1);
        ++nsubs_;
        break;
      }
      Option* p = nth_positional(positional_idx++);
      if (!p) throw ExtrasError("unexpected argument " + a);
      p->assign(a);
    }
    for (auto& o : opts_)
      if (o->required_ && !o->seen_) throw RequiredError(o->name_ + " is required");
    if (need_sub_ > 0 && nsubs_ < need_sub_) throw RequiredError("a subcommand is required");
  }
  Option* find(const std::string& key) {
    for (auto& o : opts_)
      if (o->name_ == key) return o.get();
    return nullptr;
  }
  App* find_sub(const std::string& name) {
    for (auto& s : subs_)
      if (s->name_ == name) return s.get();
    return nullptr;
  }
  Option* nth_positional(std::size_t n) {
    for (auto& o : opts_) {
      if (!o->positional()) continue;
      if (n == 0) return o.get();
      --n;
    }
    return nullptr;
  }

  std::string desc_, name_;
  std::vector<std::unique_ptr<App>> subs_;
  std::vector<std::unique_ptr<Option>> opts_;
  int need_sub_ = 0;
  int nsubs_ = 0;
  bool parsed_ = false;
};

}  // namespace CLI

#define CLI11_PARSE(app, argc, argv)      \
  try {                                   \
    (app).parse((argc), (argv));          \
  } catch (const CLI::Error& e) {         \
    return (app).exit(e);                 \
  }
