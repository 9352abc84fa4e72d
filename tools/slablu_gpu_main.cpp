// slablu_gpu — command-line front end of the B200 engine.
//
// Same verbs, config schema, validation rules, report formats and exit codes as
// the reference CLI (proj/tools/slablu_main.cpp:96-349, 353-414), driving the
// GPU engine through the C++ mirror (include/slablu_b200.hpp -> C ABI):
//   slablu_gpu solve  --config c.json [--output f] [--format csv|json] [--seed s] [--threads t]
//                     [--dump-config f]
//   slablu_gpu bench  --config c.json  (sweep_n2 + aspect; rows appended as they complete)
//   slablu_gpu verify [--quick|--full] (correctness checks re-run against the GPU factors)
// Exit codes: 0 ok, 1 config error / bad usage, 2 runtime error, 3 verification failure.
// The reference's CLI11 / nlohmann::json vendor headers are not in this image; a small
// JSON reader for the flat config objects is included here.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "slablu_b200.hpp"

namespace sb = slablu_b200;

namespace {

// ---- minimal JSON (objects, arrays, numbers, strings, booleans, null) -----------------
struct Json {
  enum Kind { Null, Bool, Int, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  int64_t i = 0;
  double d = 0.0;
  std::string s;
  std::vector<Json> a;
  std::vector<std::pair<std::string, Json>> o;  // insertion order
  bool is_int() const { return kind == Int; }
  bool is_number() const { return kind == Int || kind == Num; }
  double number() const { return kind == Int ? double(i) : d; }
  const Json* get(const std::string& k) const {
    for (auto& kv : o)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
  void set(const std::string& k, Json v) {
    for (auto& kv : o)
      if (kv.first == k) {
        kv.second = std::move(v);
        return;
      }
    o.emplace_back(k, std::move(v));
  }
};

struct Parser {
  const std::string& t;
  size_t p = 0;
  explicit Parser(const std::string& text) : t(text) {}
  [[noreturn]] void fail(const std::string& what) {
    throw sb::ConfigError("config is not valid JSON: " + what + " at offset " + std::to_string(p));
  }
  void ws() {
    while (p < t.size() && std::isspace(static_cast<unsigned char>(t[p]))) p++;
  }
  bool lit(const char* w) {
    const size_t n = strlen(w);
    if (t.compare(p, n, w) == 0) {
      p += n;
      return true;
    }
    return false;
  }
  std::string str() {
    if (t[p] != '"') fail("expected a string");
    p++;
    std::string out;
    while (p < t.size() && t[p] != '"') {
      if (t[p] == '\\') {
        p++;
        if (p >= t.size()) fail("bad escape");
        const char e = t[p];
        out += e == 'n' ? '\n' : e == 't' ? '\t' : e;
      } else {
        out += t[p];
      }
      p++;
    }
    if (p >= t.size()) fail("unterminated string");
    p++;
    return out;
  }
  Json value() {
    ws();
    if (p >= t.size()) fail("unexpected end");
    Json v;
    const char c = t[p];
    if (c == '{') {
      v.kind = Json::Obj;
      p++;
      ws();
      if (t[p] == '}') {
        p++;
        return v;
      }
      for (;;) {
        ws();
        std::string k = str();
        ws();
        if (t[p] != ':') fail("expected ':'");
        p++;
        v.o.emplace_back(k, value());
        ws();
        if (t[p] == ',') {
          p++;
          continue;
        }
        if (t[p] == '}') {
          p++;
          return v;
        }
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.kind = Json::Arr;
      p++;
      ws();
      if (t[p] == ']') {
        p++;
        return v;
      }
      for (;;) {
        v.a.push_back(value());
        ws();
        if (t[p] == ',') {
          p++;
          continue;
        }
        if (t[p] == ']') {
          p++;
          return v;
        }
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = Json::Str;
      v.s = str();
      return v;
    }
    if (lit("true")) {
      v.kind = Json::Bool;
      v.b = true;
      return v;
    }
    if (lit("false")) {
      v.kind = Json::Bool;
      return v;
    }
    if (lit("null")) return v;
    const size_t s0 = p;
    bool flt = false;
    if (t[p] == '-' || t[p] == '+') p++;
    while (p < t.size() && (std::isdigit(static_cast<unsigned char>(t[p])) || t[p] == '.' || t[p] == 'e' ||
                            t[p] == 'E' || t[p] == '-' || t[p] == '+')) {
      if (t[p] == '.' || t[p] == 'e' || t[p] == 'E') flt = true;
      p++;
    }
    if (p == s0) fail("unexpected character");
    const std::string num = t.substr(s0, p - s0);
    try {
      if (flt) {
        v.kind = Json::Num;
        v.d = std::stod(num);
      } else {
        v.kind = Json::Int;
        v.i = std::stoll(num);
      }
    } catch (...) {
      fail("bad number");
    }
    return v;
  }
  Json parse() {
    Json v = value();
    ws();
    if (p != t.size()) fail("trailing characters");
    return v;
  }
};

std::string dump(const Json& v, int indent, int level = 0) {
  const std::string pad(indent * (level + 1), ' '), pad0(indent * level, ' ');
  switch (v.kind) {
    case Json::Null: return "null";
    case Json::Bool: return v.b ? "true" : "false";
    case Json::Int: return std::to_string(v.i);
    case Json::Num: {
      char buf[40];
      std::snprintf(buf, sizeof(buf), "%.17g", v.d);
      std::string s = buf;
      if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
      return s;
    }
    case Json::Str: return "\"" + v.s + "\"";
    case Json::Arr: {
      std::string out = "[";
      for (size_t k = 0; k < v.a.size(); k++) out += (k ? ", " : "") + dump(v.a[k], indent, level + 1);
      return out + "]";
    }
    case Json::Obj: {
      std::string out = "{\n";
      for (size_t k = 0; k < v.o.size(); k++)
        out += pad + "\"" + v.o[k].first + "\": " + dump(v.o[k].second, indent, level + 1) +
               (k + 1 < v.o.size() ? ",\n" : "\n");
      return out + pad0 + "}";
    }
  }
  return "null";
}
Json jint(int64_t x) {
  Json v;
  v.kind = Json::Int;
  v.i = x;
  return v;
}
Json jnum(double x) {
  Json v;
  v.kind = Json::Num;
  v.d = x;
  return v;
}
Json jstr(const std::string& x) {
  Json v;
  v.kind = Json::Str;
  v.s = x;
  return v;
}

// ---- run configuration (slablu_main.cpp:34-189) ------------------------------------
struct RunConfig {
  std::string problem = "poisson";
  int64_t n1 = 0, n2 = 0;
  std::vector<int64_t> sweep_n2;
  double aspect = 1.0;
  std::optional<int64_t> b;
  std::optional<double> c;
  std::optional<double> kappa, ppw;
  std::string compression = "auto";
  double hbs_tol = 1e-11;
  double hbs_trunc_rel = 1e-13;
  int64_t hbs_leaf = 64;
  uint64_t seed = 0;
  int threads = 1;
  std::string format = "csv";
  std::string output;
  int device = 0;  // engine extension
};

Json load_config(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw sb::ConfigError("cannot read config file: " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  const std::string text = ss.str();
  return Parser(text).parse();
}
int64_t get_index(const Json& v, const std::string& key) {
  if (!v.is_int() || v.i < 0) throw sb::ConfigError("config key '" + key + "' must be a non-negative integer");
  return v.i;
}
double get_number(const Json& v, const std::string& key) {
  if (!v.is_number()) throw sb::ConfigError("config key '" + key + "' must be a number");
  return v.number();
}
std::string get_string(const Json& v, const std::string& key, const std::set<std::string>& allowed) {
  if (v.kind != Json::Str) throw sb::ConfigError("config key '" + key + "' must be a string");
  if (!allowed.empty() && !allowed.count(v.s)) {
    std::string msg = "config key '" + key + "' must be one of:";
    for (const auto& a : allowed) msg += " " + a;
    throw sb::ConfigError(msg);
  }
  return v.s;
}

RunConfig parse_run_config(const Json& j, bool bench) {
  if (j.kind != Json::Obj) throw sb::ConfigError("config must be a JSON object");
  static const std::set<std::string> known = {"problem", "n1", "n2", "sweep_n2", "aspect", "b", "c", "kappa", "ppw",
                                              "compression", "hbs_tol", "hbs_leaf", "seed", "hbs_trunc_rel",
                                              "threads", "format", "output", "device"};
  for (const auto& kv : j.o)
    if (!known.count(kv.first)) throw sb::ConfigError("unknown config key: " + kv.first);
  RunConfig rc;
  if (auto v = j.get("problem")) rc.problem = get_string(*v, "problem", {"poisson", "helmholtz_const", "helmholtz_varcoef"});
  if (auto v = j.get("compression")) rc.compression = get_string(*v, "compression", {"auto", "dense", "hbs"});
  if (auto v = j.get("format")) rc.format = get_string(*v, "format", {"csv", "json"});
  if (auto v = j.get("output")) rc.output = get_string(*v, "output", {});
  if (auto v = j.get("seed")) {
    if (!v->is_int() || v->i < 0) throw sb::ConfigError("config key 'seed' must be a non-negative integer");
    rc.seed = static_cast<uint64_t>(v->i);
  }
  if (auto v = j.get("threads")) {
    rc.threads = static_cast<int>(get_index(*v, "threads"));
    if (rc.threads < 1) throw sb::ConfigError("config key 'threads' must be >= 1");
  }
  if (auto v = j.get("device")) rc.device = static_cast<int>(get_index(*v, "device"));
  if (auto v = j.get("b")) rc.b = get_index(*v, "b");
  if (auto v = j.get("c")) rc.c = get_number(*v, "c");
  if (auto v = j.get("kappa")) rc.kappa = get_number(*v, "kappa");
  if (auto v = j.get("ppw")) rc.ppw = get_number(*v, "ppw");
  if (auto v = j.get("hbs_tol")) rc.hbs_tol = get_number(*v, "hbs_tol");
  if (auto v = j.get("hbs_trunc_rel")) rc.hbs_trunc_rel = get_number(*v, "hbs_trunc_rel");
  if (auto v = j.get("hbs_leaf")) rc.hbs_leaf = get_index(*v, "hbs_leaf");
  if (rc.b && rc.c) throw sb::ConfigError("set exactly one of 'b' and 'c', not both");
  if (rc.b && *rc.b < 1) throw sb::ConfigError("config key 'b' must be >= 1");
  const bool helm = rc.problem != "poisson";
  if (helm) {
    if (rc.kappa && rc.ppw) throw sb::ConfigError("set exactly one of 'kappa' and 'ppw', not both");
    if (!rc.kappa && !rc.ppw) throw sb::ConfigError("Helmholtz problems need exactly one of 'kappa' and 'ppw'");
    if (rc.kappa && *rc.kappa <= 0.0) throw sb::ConfigError("config key 'kappa' must be positive");
    if (rc.ppw && *rc.ppw <= 0.0) throw sb::ConfigError("config key 'ppw' must be positive");
  } else if (rc.kappa || rc.ppw) {
    throw sb::ConfigError("'kappa'/'ppw' apply only to Helmholtz problems");
  }
  if (bench) {
    if (j.get("n1") || j.get("n2")) throw sb::ConfigError("bench derives grids from 'sweep_n2' and 'aspect'; drop 'n1'/'n2'");
    const Json* sw = j.get("sweep_n2");
    if (!sw || sw->kind != Json::Arr || sw->a.empty())
      throw sb::ConfigError("bench needs 'sweep_n2': a non-empty array of grid sizes");
    for (const Json& v : sw->a) {
      const int64_t n2 = get_index(v, "sweep_n2");
      if (n2 < 2) throw sb::ConfigError("'sweep_n2' entries must be >= 2");
      rc.sweep_n2.push_back(n2);
    }
    if (auto v = j.get("aspect")) rc.aspect = get_number(*v, "aspect");
    if (rc.aspect < 1.0) throw sb::ConfigError("'aspect' must be >= 1 so that n1 >= n2");
  } else {
    if (j.get("sweep_n2") || j.get("aspect"))
      throw sb::ConfigError("'sweep_n2'/'aspect' are bench keys; solve takes 'n1' and 'n2'");
    if (!j.get("n1") || !j.get("n2")) throw sb::ConfigError("solve needs 'n1' and 'n2'");
    rc.n1 = get_index(*j.get("n1"), "n1");
    rc.n2 = get_index(*j.get("n2"), "n2");
    if (rc.n2 < 2 || rc.n1 < rc.n2) throw sb::ConfigError("grid must satisfy n1 >= n2 >= 2");
  }
  return rc;
}

sb::ProblemSpec make_spec(const RunConfig& rc, int64_t n1, int64_t n2) {
  if (rc.problem == "poisson") return sb::poisson_log_problem(n1, n2);
  const double kappa = rc.kappa ? *rc.kappa : sb::kappa_from_ppw(*rc.ppw, n2);
  if (rc.problem == "helmholtz_const") return sb::helmholtz_problem(n1, n2, kappa);
  return sb::helmholtz_bump_problem(n1, n2, kappa);
}

sb::SolverConfig make_solver_config(const RunConfig& rc) {
  sb::SolverConfig config;
  config.b = rc.b.value_or(0);
  if (rc.c) config.c = *rc.c;
  if (rc.compression == "dense") config.compression = sb::CompressionChoice::dense;
  else if (rc.compression == "hbs") config.compression = sb::CompressionChoice::hbs;
  config.hbs_tol = rc.hbs_tol;
  config.hbs_trunc_rel = rc.hbs_trunc_rel;
  config.hbs_leaf_size = rc.hbs_leaf;
  config.seed = rc.seed;
  config.threads = rc.threads;
  config.device = rc.device;
  return config;
}

// slablu_main.cpp:209-237: every default made explicit (a fixed point under --config)
Json resolved_config(const RunConfig& rc, bool bench) {
  Json j;
  j.kind = Json::Obj;
  j.set("problem", jstr(rc.problem));
  if (bench) {
    Json a;
    a.kind = Json::Arr;
    for (int64_t n2 : rc.sweep_n2) a.a.push_back(jint(n2));
    j.set("sweep_n2", a);
    j.set("aspect", jnum(rc.aspect));
  } else {
    j.set("n1", jint(rc.n1));
    j.set("n2", jint(rc.n2));
  }
  if (rc.b) j.set("b", jint(*rc.b));
  else j.set("c", jnum(rc.c.value_or(0.6)));
  if (rc.kappa) j.set("kappa", jnum(*rc.kappa));
  if (rc.ppw) j.set("ppw", jnum(*rc.ppw));
  j.set("compression", jstr(rc.compression));
  j.set("hbs_tol", jnum(rc.hbs_tol));
  j.set("hbs_trunc_rel", jnum(rc.hbs_trunc_rel));
  j.set("hbs_leaf", jint(rc.hbs_leaf));
  j.set("seed", jint((int64_t)rc.seed));
  j.set("threads", jint(rc.threads));
  j.set("format", jstr(rc.format));
  if (!rc.output.empty()) j.set("output", jstr(rc.output));
  if (rc.device) j.set("device", jint(rc.device));
  return j;
}

void write_text(const std::string& path, const std::string& text) {
  if (path.empty()) {
    std::cout << text << std::flush;
    return;
  }
  std::ofstream out(path);
  if (!out) throw sb::Error("cannot write output file: " + path);
  out << text;
  if (!out) throw sb::Error("failed writing output file: " + path);
}

std::string sanitize_status(std::string s) {
  for (char& ch : s)
    if (ch == ',' || ch == '\n' || ch == '"' || ch == '\\') ch = ';';
  return s;
}

int cmd_solve(const RunConfig& rc, const std::string& dump_path) {
  if (!dump_path.empty()) write_text(dump_path, dump(resolved_config(rc, false), 2) + "\n");
  const sb::SolveReport report = sb::run_problem(make_spec(rc, rc.n1, rc.n2), make_solver_config(rc));
  const std::string text = rc.format == "csv" ? std::string(sb::kCsvHeader) + "\n" + sb::csv_row(report) + "\n"
                                               : sb::json_row(report) + "\n";
  write_text(rc.output, text);
  return 0;
}

int cmd_bench(const RunConfig& rc, const std::string& dump_path) {
  if (!dump_path.empty()) write_text(dump_path, dump(resolved_config(rc, true), 2) + "\n");
  std::vector<sb::ProblemSpec> sweep;
  for (int64_t n2 : rc.sweep_n2) {
    const int64_t n1 = std::max<int64_t>(n2, static_cast<int64_t>(std::llround(rc.aspect * double(n2))));
    sweep.push_back(make_spec(rc, n1, n2));
  }
  const sb::SolverConfig config = make_solver_config(rc);
  std::ofstream file;
  std::ostream* os = &std::cout;
  if (!rc.output.empty()) {
    file.open(rc.output);
    if (!file) throw sb::Error("cannot write output file: " + rc.output);
    os = &file;
  }
  if (rc.format == "csv") {
    sb::benchmark(sweep, config, os);
    return 0;
  }
  for (const sb::ProblemSpec& spec : sweep) {  // JSON Lines, flushed per completed run
    sb::SolveReport report;
    std::string status = "ok";
    try {
      report = sb::run_problem(spec, config);
    } catch (const sb::Error& e) {
      report.n1 = spec.n1;
      report.n2 = spec.n2;
      report.n = spec.n1 * spec.n2;
      report.kappa = spec.kappa;
      report.seed = config.seed;
      status = sanitize_status(std::string("error: ") + e.what());
    }
    *os << sb::json_row(report, status.c_str()) << "\n" << std::flush;
  }
  return 0;
}

// ---- verify: correctness checks re-run against the GPU factors ---------------------------
struct Check {
  std::string name, detail;
  bool pass = false;
  double metric = 0.0;
};

// dense Gaussian elimination with partial pivoting (check reference for small grids)
std::vector<double> dense_solve(const sb::SparseSystem& s, const std::vector<double>& f) {
  const int64_t n = s.dim();
  std::vector<double> a((size_t)n * n, 0.0), x = f;
  for (int64_t r = 0; r < n; r++)
    for (int32_t p = s.row_ptr[r]; p < s.row_ptr[r + 1]; p++) a[(size_t)r * n + s.col_idx[p]] = s.values[p];
  for (int64_t k = 0; k < n; k++) {
    int64_t piv = k;
    for (int64_t r = k + 1; r < n; r++)
      if (std::fabs(a[(size_t)r * n + k]) > std::fabs(a[(size_t)piv * n + k])) piv = r;
    if (piv != k) {
      for (int64_t c = 0; c < n; c++) std::swap(a[(size_t)k * n + c], a[(size_t)piv * n + c]);
      std::swap(x[k], x[piv]);
    }
    for (int64_t r = k + 1; r < n; r++) {
      const double m = a[(size_t)r * n + k] / a[(size_t)k * n + k];
      if (m == 0.0) continue;
      for (int64_t c = k; c < n; c++) a[(size_t)r * n + c] -= m * a[(size_t)k * n + c];
      x[r] -= m * x[k];
    }
  }
  for (int64_t k = n - 1; k >= 0; k--) {
    double v = x[k];
    for (int64_t c = k + 1; c < n; c++) v -= a[(size_t)k * n + c] * x[c];
    x[k] = v / a[(size_t)k * n + k];
  }
  return x;
}

double rel_sup(const std::vector<double>& u, const std::vector<double>& ref) {
  double num = 0.0, den = 0.0;
  for (size_t k = 0; k < u.size(); k++) {
    num = std::max(num, std::fabs(u[k] - ref[k]));
    den = std::max(den, std::fabs(ref[k]));
  }
  return den > 0.0 ? num / den : num;
}

std::vector<Check> run_verification(bool full) {
  std::vector<Check> out;
  char buf[256];
  {  // elimination exactness vs dense LU on the reference's edge geometries (verify.hpp:402-428)
    double worst = 0.0;
    const int64_t geo[][3] = {{48, 48, 4}, {8, 8, 3}, {9, 8, 4}, {33, 17, 5}};
    for (auto& g : geo) {
      const sb::SparseSystem s = sb::assemble_fd5(g[0] == 33 ? sb::helmholtz_problem(g[0], g[1], 8.0)
                                                             : sb::poisson_log_problem(g[0], g[1]));
      sb::SolverConfig cfg;
      cfg.b = g[2];
      const std::vector<double> u = sb::solve(sb::factorize(s, cfg), s.rhs);
      worst = std::max(worst, rel_sup(u, dense_solve(s, s.rhs)));
    }
    std::snprintf(buf, sizeof(buf), "edge geometries vs dense LU: worst relative sup error %.2e (tol 1e-10)", worst);
    out.push_back({"elimination-exactness", buf, worst <= 1e-10, worst});
  }
  {  // discretisation golden value (test_driver.cpp:247-252)
    const sb::SparseSystem s = sb::assemble_fd5(sb::poisson_log_problem(32, 32));
    sb::SolverConfig cfg;
    cfg.b = 4;
    const std::vector<double> u = sb::solve(sb::factorize(s, cfg), s.rhs);
    const std::vector<double> ut = sb::sample_field(s, sb::poisson_log_problem(32, 32).dirichlet_data);
    const sb::ErrorReport e = sb::error_report(s, u, ut);
    const double rel = std::fabs(e.relerr_true / 4.961321e-04 - 1.0);
    std::snprintf(buf, sizeof(buf), "32x32 Poisson b=4: relerr_true %.6e (golden 4.961321e-04, rel dev %.1e)",
                  e.relerr_true, rel);
    out.push_back({"poisson-golden", buf, rel <= 1e-4, rel});
  }
  {  // factor once, solve many: bitwise repeatable (test_driver.cpp:148-161)
    const sb::SparseSystem s = sb::assemble_fd5(sb::helmholtz_bump_problem(64, 48, 30.0));
    sb::SolverConfig cfg;
    cfg.b = 6;
    const sb::Factorization f = sb::factorize(s, cfg);
    const std::vector<double> u1 = sb::solve(f, s.rhs), u2 = sb::solve(f, s.rhs);
    const bool same = u1 == u2;
    out.push_back({"determinism", same ? "repeated solves bitwise identical" : "repeated solves differ", same,
                   same ? 0.0 : 1.0});
  }
  {  // residual at direct-solver accuracy on a 10-ppw Helmholtz grid
    const int64_t n = full ? 400 : 160;
    const double kappa = sb::kappa_from_ppw(10.0, n);
    const sb::SparseSystem s = sb::assemble_fd5(sb::helmholtz_bump_problem(n, n, kappa));
    const sb::Factorization f = sb::factorize(s, sb::SolverConfig{});
    const std::vector<double> u = sb::solve(f, s.rhs);
    const sb::ErrorReport e = sb::error_report(s, u, u);
    std::snprintf(buf, sizeof(buf), "%lldx%lld bump Helmholtz 10 ppw, b=%lld: relerr_res %.2e (tol 1e-10)",
                  (long long)n, (long long)n, (long long)f.b, e.relerr_res);
    out.push_back({"residual", buf, e.relerr_res <= 1e-10, e.relerr_res});
  }
  return out;
}

int cmd_verify(bool full) {
  std::vector<Check> results;
  try {
    results = run_verification(full);
  } catch (const std::exception& e) {
    std::cerr << "verification aborted: " << e.what() << "\n";
    return 3;
  }
  size_t passed = 0;
  for (const auto& r : results) {
    std::printf("[%s] %-26s %s (metric=%.3g)\n", r.pass ? "PASS" : "FAIL", r.name.c_str(), r.detail.c_str(), r.metric);
    if (r.pass) passed++;
  }
  std::printf("verification: %zu/%zu checks passed\n", passed, results.size());
  return passed == results.size() ? 0 : 3;
}

int usage() {
  std::cerr << "slablu_gpu: two-level sparse direct solver for 2D elliptic problems (B200 engine)\n"
               "usage: slablu_gpu solve|bench --config FILE [--output FILE] [--format csv|json] [--seed N]\n"
               "                  [--threads N] [--dump-config FILE]\n"
               "       slablu_gpu verify [--quick|--full]\n";
  return 1;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage();
  const std::string verb = argv[1];
  if (verb == "--help" || verb == "-h") {
    usage();
    return 0;
  }
  if (verb != "solve" && verb != "bench" && verb != "verify") return usage();
  std::map<std::string, std::string> opt;
  bool quick = false, full = false;
  for (int k = 2; k < argc; k++) {
    const std::string a = argv[k];
    if (verb == "verify") {
      if (a == "--quick") quick = true;
      else if (a == "--full") full = true;
      else return usage();
      continue;
    }
    static const std::set<std::string> with_value = {"--config", "--output", "--format", "--seed", "--threads",
                                                     "--dump-config"};
    if (!with_value.count(a) || k + 1 >= argc) return usage();
    opt[a] = argv[++k];
  }
  if (quick && full) {
    std::cerr << "--quick excludes --full\n";
    return 1;
  }
  try {
    if (verb == "verify") return cmd_verify(full);
    if (!opt.count("--config")) return usage();
    Json j = load_config(opt["--config"]);
    if (j.kind != Json::Obj) throw sb::ConfigError("config must be a JSON object");
    if (opt.count("--seed")) j.set("seed", jint(std::stoll(opt["--seed"])));
    if (opt.count("--threads")) j.set("threads", jint(std::stoll(opt["--threads"])));
    if (opt.count("--format")) j.set("format", jstr(opt["--format"]));
    if (opt.count("--output")) j.set("output", jstr(opt["--output"]));
    const bool bench = verb == "bench";
    const RunConfig rc = parse_run_config(j, bench);
    const std::string dump_path = opt.count("--dump-config") ? opt["--dump-config"] : "";
    return bench ? cmd_bench(rc, dump_path) : cmd_solve(rc, dump_path);
  } catch (const sb::ConfigError& e) {
    std::cerr << "config error: " << e.what() << "\n";
    return 1;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }
}
