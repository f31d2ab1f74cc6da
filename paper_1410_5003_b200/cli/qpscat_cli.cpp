// qpscat — command-line front end of the B200 solver (the
// reference's `cli` module, which it never implemented: proj/tools/main.cpp:1-2).
//
//   qpscat solve    --config run.json [--out DIR] [--device N]
//   qpscat sweep    --config run.json [--out DIR] [--device N]
//   qpscat validate --config run.json
//   qpscat example  cfg1|cfg2|cfg3|cfg4|cfg5 [--seed N] [--interfaces I]   (prints a RunConfig)
//
// RunConfig (one UTF-8 JSON document):
//   { "period": 1, "omega": 10,
//     "incidence": {"theta": -0.628}
//                | {"thetas": [...]}
//                | {"uniform": {"n": 200, "lo": -3.04, "hi": -0.1}}
//                | {"alpha_grid": {"n_alpha": 40, "lo": -3.04, "hi": -0.1}},
//     "layers": [{"epsilon": 1, "mu": 1}, ...],                         (I + 1 layers)
//     "interfaces": [{"shape": "sine", "amplitude": a, "phase": p, "offset": y0, "nodes": [N]},
//                    {"shape": "polyline", "vertices": [[x, y], ...], "offset": y0, "nodes": [n1, n2, ...], "q": 6},
//                    {"shape": "fourier", "offset": y0, "cos": [...], "sin": [...], "nodes": [N]}],
//     "numerics": {"P": 60, "Mw": 40, "M": 60, "K": 0, "R": 1.5, "q": 6, "clearance": 0.75,
//                  "memory_budget": 1e12},
//     "outputs": {"residuals": true, "field_grid": {"x": [lo, hi, nx], "y": [lo, hi, ny]}} }
//
// Outputs: DIR/result.json -- the resolved config (auto K
// filled in), per-order Rayleigh-Bloch amplitudes (n, kappa, k_n, a_n,
// propagating), R, T, flux error, LSQ residual, residual suite, per-phase
// timings ("Matrix Filling / Schur Complement / Block Solve"); DIR/field.csv
// (x,y,re_u,im_u,layer) when a grid is requested; for sweeps DIR/spectra.csv
// (theta,R,T,flux_error,alpha_group,status) and DIR/sweep.json.
// Exit codes: 0 success, 2 validation failure, 3 solver
// failure, 4 memory budget exceeded, 1 anything else (device).
//
// Host code only: every computation goes through the C-ABI of
// libqpscat_b200.so (include/qpscat_b200.h).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <sys/stat.h>
#include <vector>

#include "qpscat_b200.h"

namespace {

// ----------------------------------------------------------------- JSON
struct Json {
    enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
    bool b = false;
    double num = 0;
    std::string str;
    std::vector<Json> arr;
    std::vector<std::pair<std::string, Json>> obj;
    const Json* get(const std::string& k) const {
        for (const auto& kv : obj)
            if (kv.first == k) return &kv.second;
        return nullptr;
    }
};

struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

class Parser {
public:
    explicit Parser(const std::string& s) : s_(s) {}
    Json parse() {
        Json v = value();
        ws();
        if (i_ != s_.size()) fail("trailing characters");
        return v;
    }

private:
    const std::string& s_;
    size_t i_ = 0;
    [[noreturn]] void fail(const std::string& m) {
        throw ConfigError("config: JSON " + m + " at offset " + std::to_string(i_));
    }
    void ws() {
        while (i_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[i_]))) ++i_;
    }
    bool lit(const char* w) {
        const size_t n = std::strlen(w);
        if (s_.compare(i_, n, w) == 0) {
            i_ += n;
            return true;
        }
        return false;
    }
    Json value() {
        ws();
        if (i_ >= s_.size()) fail("unexpected end");
        Json v;
        const char ch = s_[i_];
        if (ch == '{') {
            v.kind = Json::Obj;
            ++i_;
            ws();
            if (i_ < s_.size() && s_[i_] == '}') { ++i_; return v; }
            for (;;) {
                ws();
                Json k = value();
                if (k.kind != Json::Str) fail("object key must be a string");
                ws();
                if (i_ >= s_.size() || s_[i_] != ':') fail("expected ':'");
                ++i_;
                v.obj.emplace_back(k.str, value());
                ws();
                if (i_ < s_.size() && s_[i_] == ',') { ++i_; continue; }
                if (i_ < s_.size() && s_[i_] == '}') { ++i_; return v; }
                fail("expected ',' or '}'");
            }
        }
        if (ch == '[') {
            v.kind = Json::Arr;
            ++i_;
            ws();
            if (i_ < s_.size() && s_[i_] == ']') { ++i_; return v; }
            for (;;) {
                v.arr.push_back(value());
                ws();
                if (i_ < s_.size() && s_[i_] == ',') { ++i_; continue; }
                if (i_ < s_.size() && s_[i_] == ']') { ++i_; return v; }
                fail("expected ',' or ']'");
            }
        }
        if (ch == '"') {
            v.kind = Json::Str;
            ++i_;
            while (i_ < s_.size() && s_[i_] != '"') {
                if (s_[i_] == '\\' && i_ + 1 < s_.size()) ++i_;
                v.str.push_back(s_[i_++]);
            }
            if (i_ >= s_.size()) fail("unterminated string");
            ++i_;
            return v;
        }
        if (lit("true")) { v.kind = Json::Bool; v.b = true; return v; }
        if (lit("false")) { v.kind = Json::Bool; v.b = false; return v; }
        if (lit("null")) return v;
        char* end = nullptr;
        v.num = std::strtod(s_.c_str() + i_, &end);
        if (end == s_.c_str() + i_) fail("bad value");
        i_ = size_t(end - s_.c_str());
        v.kind = Json::Num;
        return v;
    }
};

std::string fmt(double x) {
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", x);
    return b;
}

// ------------------------------------------------------------- run config
struct Iface {
    std::string shape = "sine";
    double amplitude = 0, phase = 0, offset = 0;
    std::vector<double> cosc, sinc, verts;  // verts: x0,y0,x1,y1,...
    std::vector<int> nodes;
    int q = 6;
};

struct RunConfig {
    double d = 1.0, omega = 0;
    std::string inc_kind = "theta";
    std::vector<double> thetas;
    int grid_n = 0;
    double lo = 0, hi = 0;
    std::vector<double> eps, mu;
    std::vector<Iface> ifaces;
    qps_numerics num{60, 120, 60, 0, 2.0, 6, 0.05, uint64_t(4) << 30};
    bool residuals = false;
    bool field = false;
    double fx[3] = {0, 0, 0}, fy[3] = {0, 0, 0};
};

double need_num(const Json& o, const char* k, const std::string& path) {
    const Json* v = o.get(k);
    if (!v || v->kind != Json::Num) throw ConfigError("config: " + path + "." + k + " missing or not a number");
    return v->num;
}
double opt_num(const Json& o, const char* k, double def) {
    const Json* v = o.get(k);
    return (v && v->kind == Json::Num) ? v->num : def;
}
std::vector<double> num_array(const Json* v, const std::string& path) {
    std::vector<double> out;
    if (!v) return out;
    if (v->kind != Json::Arr) throw ConfigError("config: " + path + " must be an array");
    for (const auto& e : v->arr) {
        if (e.kind != Json::Num) throw ConfigError("config: " + path + " must hold numbers");
        out.push_back(e.num);
    }
    return out;
}

RunConfig read_config(const Json& j) {
    if (j.kind != Json::Obj) throw ConfigError("config: top level must be an object");
    RunConfig c;
    c.d = opt_num(j, "period", 1.0);
    c.omega = need_num(j, "omega", "");
    const Json* inc = j.get("incidence");
    if (!inc || inc->kind != Json::Obj) throw ConfigError("config: incidence missing");
    if (const Json* t = inc->get("theta")) {
        c.inc_kind = "theta";
        if (t->kind != Json::Num) throw ConfigError("config: incidence.theta must be a number");
        c.thetas = {t->num};
    } else if (inc->get("thetas")) {
        c.inc_kind = "thetas";
        c.thetas = num_array(inc->get("thetas"), "incidence.thetas");
    } else if (const Json* u = inc->get("uniform")) {
        c.inc_kind = "uniform";
        c.grid_n = int(need_num(*u, "n", "incidence.uniform"));
        c.lo = need_num(*u, "lo", "incidence.uniform");
        c.hi = need_num(*u, "hi", "incidence.uniform");
        for (int a = 0; a < c.grid_n; ++a)
            c.thetas.push_back(c.grid_n > 1 ? c.lo + (c.hi - c.lo) * a / (c.grid_n - 1) : c.lo);
    } else if (const Json* g = inc->get("alpha_grid")) {
        c.inc_kind = "alpha_grid";
        c.grid_n = int(need_num(*g, "n_alpha", "incidence.alpha_grid"));
        c.lo = need_num(*g, "lo", "incidence.alpha_grid");
        c.hi = need_num(*g, "hi", "incidence.alpha_grid");
    } else {
        throw ConfigError("config: incidence needs theta, thetas, uniform or alpha_grid");
    }
    const Json* layers = j.get("layers");
    if (!layers || layers->kind != Json::Arr) throw ConfigError("config: layers missing");
    for (size_t i = 0; i < layers->arr.size(); ++i) {
        const std::string p = "layers[" + std::to_string(i) + "]";
        c.eps.push_back(need_num(layers->arr[i], "epsilon", p));
        c.mu.push_back(opt_num(layers->arr[i], "mu", 1.0));
    }
    const Json* ifs = j.get("interfaces");
    if (!ifs || ifs->kind != Json::Arr) throw ConfigError("config: interfaces missing");
    for (size_t i = 0; i < ifs->arr.size(); ++i) {
        const Json& e = ifs->arr[i];
        const std::string p = "interfaces[" + std::to_string(i) + "]";
        Iface f;
        const Json* sh = e.get("shape");
        f.shape = sh && sh->kind == Json::Str ? sh->str : "sine";
        f.offset = opt_num(e, "offset", 0.0);
        f.amplitude = opt_num(e, "amplitude", 0.0);
        f.phase = opt_num(e, "phase", 0.0);
        f.q = int(opt_num(e, "q", 6));
        f.cosc = num_array(e.get("cos"), p + ".cos");
        f.sinc = num_array(e.get("sin"), p + ".sin");
        for (double v : num_array(e.get("nodes"), p + ".nodes")) f.nodes.push_back(int(v));
        if (const Json* vs = e.get("vertices")) {
            if (vs->kind != Json::Arr) throw ConfigError("config: " + p + ".vertices must be an array");
            for (const auto& xy : vs->arr) {
                const auto v = num_array(&xy, p + ".vertices[]");
                if (v.size() != 2) throw ConfigError("config: " + p + ".vertices entries are [x, y]");
                f.verts.push_back(v[0]);
                f.verts.push_back(v[1]);
            }
        }
        if (f.shape != "sine" && f.shape != "polyline" && f.shape != "fourier")
            throw ConfigError("config: " + p + ".shape must be sine, polyline or fourier");
        if (f.nodes.empty()) throw ConfigError("config: " + p + ".nodes missing");
        c.ifaces.push_back(f);
    }
    if (const Json* n = j.get("numerics")) {
        c.num.P = int(opt_num(*n, "P", c.num.P));
        c.num.Mw = int(opt_num(*n, "Mw", c.num.Mw));
        c.num.M = int(opt_num(*n, "M", c.num.M));
        c.num.K = int(opt_num(*n, "K", c.num.K));
        c.num.R = opt_num(*n, "R", c.num.R);
        c.num.grading_q = int(opt_num(*n, "q", c.num.grading_q));
        c.num.clearance = opt_num(*n, "clearance", c.num.clearance);
        c.num.memory_budget = uint64_t(opt_num(*n, "memory_budget", double(c.num.memory_budget)));
    }
    if (const Json* o = j.get("outputs")) {
        if (const Json* r = o->get("residuals")) c.residuals = r->kind == Json::Bool && r->b;
        if (const Json* g = o->get("field_grid")) {
            const auto x = num_array(g->get("x"), "outputs.field_grid.x");
            const auto y = num_array(g->get("y"), "outputs.field_grid.y");
            if (x.size() != 3 || y.size() != 3) throw ConfigError("config: field_grid x / y are [lo, hi, n]");
            c.field = true;
            for (int k = 0; k < 3; ++k) {
                c.fx[k] = x[k];
                c.fy[k] = y[k];
            }
        }
    }
    return c;
}

std::string config_json(const RunConfig& c, int K_resolved) {
    std::ostringstream o;
    o << "{\n  \"period\": " << fmt(c.d) << ",\n  \"omega\": " << fmt(c.omega) << ",\n  \"incidence\": ";
    if (c.inc_kind == "theta") {
        o << "{\"theta\": " << fmt(c.thetas.at(0)) << "}";
    } else if (c.inc_kind == "thetas") {
        o << "{\"thetas\": [";
        for (size_t a = 0; a < c.thetas.size(); ++a) o << (a ? ", " : "") << fmt(c.thetas[a]);
        o << "]}";
    } else {
        o << "{\"" << c.inc_kind << "\": {\"" << (c.inc_kind == "uniform" ? "n" : "n_alpha") << "\": " << c.grid_n
          << ", \"lo\": " << fmt(c.lo) << ", \"hi\": " << fmt(c.hi) << "}}";
    }
    o << ",\n  \"layers\": [";
    for (size_t i = 0; i < c.eps.size(); ++i)
        o << (i ? ", " : "") << "{\"epsilon\": " << fmt(c.eps[i]) << ", \"mu\": " << fmt(c.mu[i]) << "}";
    o << "],\n  \"interfaces\": [";
    for (size_t i = 0; i < c.ifaces.size(); ++i) {
        const Iface& f = c.ifaces[i];
        o << (i ? ",\n    " : "\n    ") << "{\"shape\": \"" << f.shape << "\", \"offset\": " << fmt(f.offset);
        if (f.shape == "sine") o << ", \"amplitude\": " << fmt(f.amplitude) << ", \"phase\": " << fmt(f.phase);
        if (f.shape == "fourier") {
            o << ", \"cos\": [";
            for (size_t m = 0; m < f.cosc.size(); ++m) o << (m ? ", " : "") << fmt(f.cosc[m]);
            o << "], \"sin\": [";
            for (size_t m = 0; m < f.sinc.size(); ++m) o << (m ? ", " : "") << fmt(f.sinc[m]);
            o << "]";
        }
        if (f.shape == "polyline") {
            o << ", \"vertices\": [";
            for (size_t m = 0; m < f.verts.size(); m += 2)
                o << (m ? ", " : "") << "[" << fmt(f.verts[m]) << ", " << fmt(f.verts[m + 1]) << "]";
            o << "], \"q\": " << f.q;
        }
        o << ", \"nodes\": [";
        for (size_t m = 0; m < f.nodes.size(); ++m) o << (m ? ", " : "") << f.nodes[m];
        o << "]}";
    }
    o << "],\n  \"numerics\": {\"P\": " << c.num.P << ", \"Mw\": " << c.num.Mw << ", \"M\": " << c.num.M
      << ", \"K\": " << K_resolved << ", \"R\": " << fmt(c.num.R) << ", \"q\": " << c.num.grading_q
      << ", \"clearance\": " << fmt(c.num.clearance) << ", \"memory_budget\": " << c.num.memory_budget << "}";
    if (c.residuals || c.field) {
        o << ",\n  \"outputs\": {\"residuals\": " << (c.residuals ? "true" : "false");
        if (c.field)
            o << ", \"field_grid\": {\"x\": [" << fmt(c.fx[0]) << ", " << fmt(c.fx[1]) << ", " << fmt(c.fx[2])
              << "], \"y\": [" << fmt(c.fy[0]) << ", " << fmt(c.fy[1]) << ", " << fmt(c.fy[2]) << "]}";
        o << "}";
    }
    o << "\n}";
    return o.str();
}

// ------------------------------------------------------ built-in examples
// BASELINE.json configs 1-5, the generator of paper_1410_5003_b200/configs.py
// (std::mt19937_64(seed), u = (x >> 11) 2^-53, draws per interface then per
// layer; omega = k_1, eps_i = (k_i / k_1)^2).
struct Rng {
    std::mt19937_64 g;
    explicit Rng(uint64_t s) : g(s) {}
    double u(double lo = 0.0, double hi = 1.0) { return lo + (hi - lo) * (double(g() >> 11) * 0x1.0p-53); }
};

RunConfig example(int cfg, uint64_t seed, int nif) {
    const double pi = 3.14159265358979323846;
    RunConfig c;
    Rng r(seed);
    std::vector<double> ks;
    auto sine = [](double off, double a, double phi, int N) {
        Iface f;
        f.shape = "sine";
        f.offset = off;
        f.amplitude = a;
        f.phase = phi;
        f.nodes = {N};
        return f;
    };
    c.num = qps_numerics{60, 40, 60, 10, 1.5, 6, 0.75, uint64_t(1) << 40};
    if (cfg == 1) {
        ks = {10.0, 15.0};
        c.ifaces.push_back(sine(0.0, 0.25, 0.0, 80));
        c.thetas = {-pi / 5};
    } else if (cfg == 2 || cfg == 4 || cfg == 5) {
        int I = cfg == 2 ? 10 : cfg == 4 ? 1000 : 100;
        const int N = cfg == 2 ? 100 : cfg == 4 ? 300 : 150;
        if (nif > 0) I = nif;
        for (int i = 0; i < I; ++i) {
            const double a = r.u(0.05, 0.3);
            const double phi = r.u(0.0, 2 * pi);
            c.ifaces.push_back(sine(-1.0 * i, a, phi, N));
        }
        for (int i = 0; i <= I; ++i) ks.push_back(cfg == 2 ? 10.0 * r.u(1.0, 3.0) : r.u(10.0, 30.0));
        c.num.P = cfg == 4 ? 80 : 60;
        c.num.K = cfg == 2 ? 10 : 20;
        c.thetas = {-pi / 5};
    } else if (cfg == 3) {
        const int I = nif > 0 ? nif : 100;
        const double top = 0.5 * (I - 1);
        for (int i = 0; i < I; ++i) {
            if (i % 2 == 0) {
                const double a = r.u(0.05, 0.3);
                const double phi = r.u(0.0, 2 * pi);
                c.ifaces.push_back(sine(top - 1.0 * i, a, phi, 200));
            } else {
                const bool trapezoid = r.u() >= 0.5;
                const double h = r.u(0.1, 0.3);
                Iface f;
                f.shape = "polyline";
                f.offset = top - 1.0 * i;
                if (trapezoid) {
                    const double x1 = r.u(-0.3, -0.1), x2 = r.u(0.1, 0.3);
                    f.verts = {-0.5, 0.0, x1, h, x2, h, 0.5, 0.0};
                } else {
                    const double xl = r.u(-0.3, -0.1), xp = r.u(0.0, 0.2);
                    f.verts = {-0.5, 0.0, xl, 0.0, xp, h, 0.5, 0.0};
                }
                f.nodes = {67, 67, 66};
                f.q = 6;
                c.ifaces.push_back(f);
            }
        }
        for (int i = 0; i <= I; ++i) ks.push_back(10.0 * r.u(1.0, 3.0));
        c.thetas = {-std::acos(-1.0 + 2.0 * pi / ks[0]) + 1e-10};
    } else {
        throw ConfigError("example: config must be cfg1 .. cfg5");
    }
    c.omega = ks[0];
    for (double k : ks) {
        c.eps.push_back((k / ks[0]) * (k / ks[0]));
        c.mu.push_back(1.0);
    }
    c.inc_kind = "theta";
    if (cfg == 5) {
        c.inc_kind = "uniform";
        c.grid_n = 200;
        c.lo = -pi + 0.1;
        c.hi = -0.1;
        c.thetas.clear();
        for (int a = 0; a < 200; ++a) c.thetas.push_back(c.lo + (c.hi - c.lo) * a / 199);
    }
    return c;
}

// --------------------------------------------------------------- running
struct Lib {
    qps_ctx* h = nullptr;
    ~Lib() { qps_destroy(h); }
};

struct Failure : std::runtime_error {
    int code;
    Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void check(qps_ctx* h, int st) {
    if (st == QPS_OK) return;
    char msg[1024] = {0};
    int layer = 0;
    uint64_t bytes = 0;
    qps_last_error(h, msg, sizeof msg, &layer, &bytes);
    int code = 1;
    switch (st) {
        case QPS_ERR_CONFIG: case QPS_ERR_GEOMETRY: case QPS_ERR_USAGE: case QPS_ERR_DOMAIN: code = 2; break;
        case QPS_ERR_SOLVER: case QPS_ERR_SINGULARITY: code = 3; break;
        case QPS_ERR_MEMORY_BUDGET: code = 4; break;
        default: code = 1;
    }
    std::string m = msg;
    if (st == QPS_ERR_SOLVER) m += " (layer " + std::to_string(layer) + ")";
    if (st == QPS_ERR_MEMORY_BUDGET) m += " (" + std::to_string(bytes) + " bytes required)";
    throw Failure(code, m);
}

void setup(qps_ctx* h, const RunConfig& c, double theta) {
    const int I = int(c.ifaces.size());
    std::vector<qps_interface_spec> specs(I);
    for (int j = 0; j < I; ++j) {
        const Iface& f = c.ifaces[j];
        qps_interface_spec& s = specs[j];
        s = qps_interface_spec{};
        s.shape = f.shape == "sine" ? QPS_SHAPE_SINE : f.shape == "fourier" ? QPS_SHAPE_FOURIER : QPS_SHAPE_POLYLINE;
        s.offset = f.offset;
        s.amplitude = f.amplitude;
        s.phase = f.phase;
        s.n_cos = int(f.cosc.size());
        s.cosc = f.cosc.data();
        s.n_sin = int(f.sinc.size());
        s.sinc = f.sinc.data();
        s.n_vertices = int(f.verts.size() / 2);
        s.vertices = f.verts.data();
        s.n_nodes = int(f.nodes.size());
        s.nodes = f.nodes.data();
        s.grading_q = f.q;
    }
    check(h, qps_build_geometry(h, c.d, int(c.eps.size()), c.eps.data(), c.mu.data(), I, specs.data(), &c.num));
    check(h, qps_make_problem(h, c.omega, theta, c.num.K));
}

void write_file(const std::string& path, const std::string& text) {
    std::ofstream f(path);
    if (!f) throw Failure(1, "cannot write " + path);
    f << text;
}

std::string cx(qps_cplx z) { return "[" + fmt(z.re) + ", " + fmt(z.im) + "]"; }

int run_solve(const RunConfig& c, const std::string& out, int device) {
    if (c.thetas.size() != 1) throw ConfigError("solve: incidence must be a single theta (use `sweep` for lists)");
    Lib L;
    L.h = qps_create(device);
    if (!L.h) throw Failure(1, "no usable CUDA device");
    setup(L.h, c, c.thetas[0]);
    check(L.h, qps_solve(L.h));
    int I = 0, K = 0;
    check(L.h, qps_problem_info(L.h, &I, &K, nullptr, nullptr, nullptr, nullptr, nullptr));
    const int nrb = 2 * K + 1;
    std::vector<double> kappa(nrb);
    std::vector<qps_cplx> kU(nrb), kD(nrb), aU(nrb), aD(nrb);
    std::vector<int> pu(nrb), pd(nrb);
    double R = 0, T = 0, fe = 0, mx = 0;
    check(L.h, qps_reflection_transmission(L.h, &R, &T, &fe, kappa.data(), kU.data(), kD.data(), pu.data(), pd.data()));
    check(L.h, qps_get_solution(L.h, nullptr, nullptr, aU.data(), aD.data(), nullptr, &mx));
    qps_phase_times t{};
    check(L.h, qps_get_phase_times(L.h, &t));
    std::ostringstream o;
    o << "{\n\"config\": " << config_json(c, K) << ",\n\"R\": " << fmt(R) << ",\n\"T\": " << fmt(T)
      << ",\n\"flux_error\": " << fmt(fe) << ",\n\"max_lsq_residual\": " << fmt(mx) << ",\n\"timings_ms\": {"
      << "\"matrix_filling\": " << fmt(t.fill_ms + t.assemble_ms) << ", \"schur_complement\": " << fmt(t.schur_ms)
      << ", \"block_solve\": " << fmt(t.solve_ms + t.recover_ms) << ", \"total_device\": " << fmt(t.total_ms)
      << "},\n\"orders\": [";
    for (int i = 0; i < nrb; ++i)
        o << (i ? ",\n  " : "\n  ") << "{\"n\": " << i - K << ", \"kappa\": " << fmt(kappa[i]) << ", \"kU\": "
          << cx(kU[i]) << ", \"aU\": " << cx(aU[i]) << ", \"propagating_up\": " << (pu[i] ? "true" : "false")
          << ", \"kD\": " << cx(kD[i]) << ", \"aD\": " << cx(aD[i])
          << ", \"propagating_down\": " << (pd[i] ? "true" : "false") << "}";
    o << "]";
    if (c.residuals) {
        std::vector<int> probe;
        for (int j : {0, I / 2, I - 1})
            if (probe.empty() || probe.back() != j) probe.push_back(j);
        double w = 0, r = 0, itf = 0;
        check(L.h, qps_residual_suite(L.h, int(probe.size()), probe.data(), &w, &r, &itf));
        o << ",\n\"residuals\": {\"wall_qp\": " << fmt(w) << ", \"radiation\": " << fmt(r)
          << ", \"interface\": " << fmt(itf) << "}";
    }
    if (c.field) {
        const int nx = int(c.fx[2]), ny = int(c.fy[2]);
        std::vector<double> xy;
        for (int b = 0; b < ny; ++b)
            for (int a = 0; a < nx; ++a) {
                xy.push_back(nx > 1 ? c.fx[0] + (c.fx[1] - c.fx[0]) * a / (nx - 1) : c.fx[0]);
                xy.push_back(ny > 1 ? c.fy[0] + (c.fy[1] - c.fy[0]) * b / (ny - 1) : c.fy[0]);
            }
        const int n = nx * ny;
        std::vector<qps_cplx> u(n);
        std::vector<int> lay(n), reg(n);
        check(L.h, qps_evaluate_field(L.h, n, xy.data(), nullptr, u.data(), reg.data(), lay.data()));
        std::ostringstream f;
        f << "x,y,re_u,im_u,layer\n";
        for (int i = 0; i < n; ++i)
            f << fmt(xy[2 * i]) << "," << fmt(xy[2 * i + 1]) << "," << fmt(u[i].re) << "," << fmt(u[i].im) << ","
              << (reg[i] == 1 ? lay[i] : reg[i] == 0 ? -1 : I + 1) << "\n";
        write_file(out + "/field.csv", f.str());
        o << ",\n\"field_csv\": \"field.csv\"";
    }
    o << "\n}\n";
    write_file(out + "/result.json", o.str());
    std::printf("R = %.15g  T = %.15g  flux error = %.3e  (device %.1f ms)\n", R, T, fe, t.total_ms);
    return 0;
}

int run_sweep(const RunConfig& c, const std::string& out, int device) {
    Lib L;
    L.h = qps_create(device);
    if (!L.h) throw Failure(1, "no usable CUDA device");
    std::vector<double> th = c.thetas;
    setup(L.h, c, th.empty() ? -1.0 : th[0]);
    if (c.inc_kind == "alpha_grid") {
        int n = 0;
        check(L.h, qps_plan_sweep(L.h, c.grid_n, c.lo, c.hi, 0, nullptr, nullptr, &n));
        th.assign(n, 0.0);
        check(L.h, qps_plan_sweep(L.h, c.grid_n, c.lo, c.hi, n, th.data(), nullptr, &n));
        check(L.h, qps_make_problem(L.h, c.omega, th.at(0), c.num.K));
    }
    int I = 0, K = 0;
    check(L.h, qps_problem_info(L.h, &I, &K, nullptr, nullptr, nullptr, nullptr, nullptr));
    const int n = int(th.size()), nrb = 2 * K + 1;
    std::vector<double> R(n), T(n), fe(n);
    std::vector<qps_cplx> aU(size_t(n) * nrb), aD(size_t(n) * nrb);
    std::vector<int> st(n), grp(n);
    check(L.h, qps_sweep(L.h, n, th.data(), K, 0, R.data(), T.data(), fe.data(), aU.data(), aD.data(), st.data()));
    int ng = 0;
    uint64_t ni = 0, nf = 0;
    check(L.h, qps_sweep_info(L.h, n, grp.data(), &ng, &ni, &nf));
    qps_phase_times t{};
    check(L.h, qps_get_phase_times(L.h, &t));
    std::ostringstream csv;
    csv << "theta,R,T,flux_error,alpha_group,status\n";
    double mean_fe = 0;
    int ok = 0;
    for (int a = 0; a < n; ++a) {
        csv << fmt(th[a]) << "," << fmt(R[a]) << "," << fmt(T[a]) << "," << fmt(fe[a]) << "," << grp[a] << ","
            << st[a] << "\n";
        if (st[a] == QPS_OK) {
            mean_fe += std::abs(fe[a]);
            ++ok;
        }
    }
    write_file(out + "/spectra.csv", csv.str());
    std::ostringstream o;
    o << "{\n\"config\": " << config_json(c, K) << ",\n\"angles\": " << n << ",\n\"solved\": " << ok
      << ",\n\"alpha_groups\": " << ng << ",\n\"interior_eliminations\": " << ni << ",\n\"factorizations\": " << nf
      << ",\n\"mean_abs_flux_error\": " << fmt(ok ? mean_fe / ok : NAN) << ",\n\"timings_ms\": {\"total_device\": "
      << fmt(t.total_ms) << ", \"matrix_filling\": " << fmt(t.fill_ms + t.assemble_ms) << ", \"schur_complement\": "
      << fmt(t.schur_ms) << ", \"block_solve\": " << fmt(t.solve_ms + t.recover_ms) << "},\n\"spectra_csv\": \"spectra.csv\"\n}\n";
    write_file(out + "/sweep.json", o.str());
    std::printf("%d/%d angles solved, %d alpha groups, %llu factorizations, %.1f ms\n", ok, n, ng,
                (unsigned long long)nf, t.total_ms);
    return ok == n ? 0 : 3;
}

int run_validate(const RunConfig& c) {
    Lib L;
    L.h = qps_create(-1);  // host-only context: geometry and problem setup, no device work
    if (!L.h) throw Failure(1, "cannot create a context");
    setup(L.h, c, c.thetas.empty() ? -1.0 : c.thetas[0]);
    int I = 0, K = 0;
    check(L.h, qps_problem_info(L.h, &I, &K, nullptr, nullptr, nullptr, nullptr, nullptr));
    std::printf("valid: %d interfaces, K = %d\n", I, K);
    return 0;
}

void usage() {
    std::fprintf(stderr,
                 "usage: qpscat solve|sweep|validate --config FILE [--out DIR] [--device N]\n"
                 "       qpscat example cfg1..cfg5 [--seed N] [--interfaces I]\n");
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        return 2;
    }
    const std::string cmd = argv[1];
    std::map<std::string, std::string> opt;
    std::vector<std::string> pos;
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        if (a.rfind("--", 0) == 0 && i + 1 < argc) opt[a.substr(2)] = argv[++i];
        else pos.push_back(a);
    }
    try {
        if (cmd == "example") {
            if (pos.empty()) throw ConfigError("example: which config (cfg1 .. cfg5)?");
            const int cfg = pos[0].size() == 4 ? pos[0][3] - '0' : 0;
            const RunConfig c = example(cfg, opt.count("seed") ? std::stoull(opt["seed"]) : 5003,
                                        opt.count("interfaces") ? std::stoi(opt["interfaces"]) : 0);
            std::printf("%s\n", config_json(c, c.num.K).c_str());
            return 0;
        }
        if (!opt.count("config")) throw ConfigError("--config FILE required");
        std::ifstream f(opt["config"]);
        if (!f) throw ConfigError("cannot read " + opt["config"]);
        std::stringstream ss;
        ss << f.rdbuf();
        const RunConfig c = read_config(Parser(ss.str()).parse());
        const std::string out = opt.count("out") ? opt["out"] : ".";
        ::mkdir(out.c_str(), 0755);
        const int device = opt.count("device") ? std::stoi(opt["device"]) : 0;
        if (cmd == "solve") return run_solve(c, out, device);
        if (cmd == "sweep") return run_sweep(c, out, device);
        if (cmd == "validate") return run_validate(c);
        usage();
        return 2;
    } catch (const ConfigError& e) {
        std::fprintf(stderr, "qpscat: %s\n", e.what());
        return 2;
    } catch (const Failure& e) {
        std::fprintf(stderr, "qpscat: %s\n", e.what());
        return e.code;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "qpscat: %s\n", e.what());
        return 1;
    }
}
