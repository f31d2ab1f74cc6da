// ORACLE TEST INFRASTRUCTURE — not product code.
//
// include/qpscat_b200.h implemented by the REFERENCE itself: the qpscat
// headers (/root/reference/proj/include/qpscat) compiled unmodified against
// oracle/shim.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs load the resulting
// oracle/_ref/libqpscat_ref.so, always as the checker or the CPU baseline.
// Every entry point is a direct call sequence into the reference API; the
// composition mirrors the reference's own drivers (proj/tests/test_tridiag.cpp:
// 112-126 `solve_stack`, proj/tests/test_assembly.cpp:229-239 for re-assembly).
#include <chrono>
#include <cstring>
#include <memory>
#include <optional>
#include <string>

#include "qpscat/postprocess.hpp"
#include "qpscat_b200.h"

using namespace qpscat;

struct qps_ctx {
    LayerStack stack;
    NumericsParams num;
    StackGeometry geom;
    ScatteringProblem prob;
    bool have_geom = false, have_prob = false;
    std::optional<ShiftBlockCache> cache;
    std::optional<BlockSystem> sys;
    std::optional<PeriodizedSystem> ps;
    std::vector<Vec> eta;
    std::optional<Solution> sol;
    qps_phase_times times{};
    uint64_t fill_evals = 0;
    std::string err;
    int err_layer = 0;
    uint64_t err_bytes = 0;
    // last sweep: alpha group per angle, interior eliminations, block factorizations
    std::vector<int> sweep_group;
    int sweep_ngroups = 0;
    uint64_t sweep_interior = 0, sweep_factorizations = 0;
};

namespace {

using clk = std::chrono::steady_clock;
double ms_since(clk::time_point t0) {
    return std::chrono::duration<double, std::milli>(clk::now() - t0).count();
}

template <class F>
int guarded(qps_ctx* c, F&& f) {
    if (!c) return QPS_ERR_USAGE;
    c->err.clear();
    c->err_layer = 0;
    c->err_bytes = 0;
    try {
        f();
        return QPS_OK;
    } catch (const SolverError& e) {
        c->err = e.what();
        c->err_layer = e.layer;
        return QPS_ERR_SOLVER;
    } catch (const MemoryBudgetError& e) {
        c->err = e.what();
        c->err_bytes = e.required_bytes;
        return QPS_ERR_MEMORY_BUDGET;
    } catch (const ConfigError& e) {
        c->err = e.what();
        return QPS_ERR_CONFIG;
    } catch (const GeometryError& e) {
        c->err = e.what();
        return QPS_ERR_GEOMETRY;
    } catch (const UsageError& e) {
        c->err = e.what();
        return QPS_ERR_USAGE;
    } catch (const SingularityError& e) {
        c->err = e.what();
        return QPS_ERR_SINGULARITY;
    } catch (const std::domain_error& e) {
        c->err = e.what();
        return QPS_ERR_DOMAIN;
    } catch (const std::exception& e) {
        c->err = e.what();
        return QPS_ERR_INTERNAL;
    }
}

void need(bool ok, const char* what) {
    if (!ok) throw UsageError(std::string("qps oracle: ") + what);
}

void put(const Mat& m, qps_cplx* out, int* rows, int* cols) {
    if (rows) *rows = int(m.rows());
    if (cols) *cols = int(m.cols());
    if (out && m.size()) std::memcpy(out, m.data(), sizeof(cd) * m.size());
}

const Mat& pick(const std::vector<Mat>& v, int i) {
    if (i < 0 || i >= int(v.size())) throw UsageError("qps oracle: block index out of range");
    return v[i];
}

}  // namespace

extern "C" {

int qps_abi_version(void) { return QPS_ABI_VERSION; }
const char* qps_backend_name(void) { return "reference-cpu"; }

qps_ctx* qps_create(int) { return new qps_ctx(); }
void qps_destroy(qps_ctx* c) { delete c; }

int qps_last_error(const qps_ctx* c, char* msg, size_t cap, int* layer, uint64_t* bytes) {
    if (!c) return QPS_ERR_USAGE;
    if (msg && cap) {
        std::strncpy(msg, c->err.c_str(), cap - 1);
        msg[cap - 1] = 0;
    }
    if (layer) *layer = c->err_layer;
    if (bytes) *bytes = c->err_bytes;
    return QPS_OK;
}

int qps_set_num_threads(qps_ctx* c, int n) {
    return guarded(c, [&] {
        set_num_threads(n);
        if (n > 0) qps_blas::set_num_threads(n);
    });
}

int qps_set_qsolve_threshold(qps_ctx* c, double th) {
    return guarded(c, [&] { qsolve_threshold() = th; });
}

// product extension (iterative refinement of the GPU's cyclic reduction): the
// reference's block Thomas has nothing to refine
int qps_set_refine(qps_ctx* c, int steps) { return (c && steps >= -1 && steps <= 4) ? QPS_OK : QPS_ERR_USAGE; }

int qps_build_geometry(qps_ctx* c, double d, int n_layers, const double* eps, const double* mu, int n_ifaces,
                       const qps_interface_spec* ifs, const qps_numerics* num) {
    return guarded(c, [&] {
        need(num != nullptr, "numerics required");
        c->have_geom = c->have_prob = false;
        c->cache.reset();
        c->sys.reset();
        c->ps.reset();
        c->sol.reset();
        LayerStack st;
        st.d = d;
        for (int i = 0; i < n_layers; ++i) st.materials.push_back({eps[i], mu ? mu[i] : 1.0});
        for (int j = 0; j < n_ifaces; ++j) {
            const auto& s = ifs[j];
            InterfaceSpec sp;
            sp.shape = s.shape == QPS_SHAPE_SINE      ? InterfaceSpec::Shape::Sine
                       : s.shape == QPS_SHAPE_FOURIER ? InterfaceSpec::Shape::Fourier
                                                      : InterfaceSpec::Shape::Polyline;
            sp.offset = s.offset;
            sp.amplitude = s.amplitude;
            sp.phase = s.phase;
            sp.cosc.assign(s.cosc, s.cosc + s.n_cos);
            sp.sinc.assign(s.sinc, s.sinc + s.n_sin);
            for (int v = 0; v < s.n_vertices; ++v) sp.vertices.push_back({s.vertices[2 * v], s.vertices[2 * v + 1]});
            sp.nodes.assign(s.nodes, s.nodes + s.n_nodes);
            sp.grading_q = s.grading_q;
            st.interfaces.push_back(std::move(sp));
        }
        NumericsParams np;
        np.P = num->P;
        np.Mw = num->Mw;
        np.M = num->M;
        np.K = num->K;
        np.R = num->R;
        np.grading_q = num->grading_q;
        np.clearance = num->clearance;
        np.memory_budget = num->memory_budget;
        c->stack = std::move(st);
        c->num = np;
        c->geom = build_geometry(c->stack, c->num);
        c->have_geom = true;
    });
}

int qps_make_problem(qps_ctx* c, double omega, double theta, int K) {
    return guarded(c, [&] {
        need(c->have_geom, "build_geometry first");
        c->prob = make_problem(c->stack, c->geom, omega, theta, K);
        c->have_prob = true;
        c->sys.reset();
        c->ps.reset();
        c->sol.reset();
    });
}

int qps_problem_info(const qps_ctx* c, int* I, int* K, int* n_nodes, double* k, qps_cplx* alpha, double* y_U,
                     double* y_D) {
    return guarded(const_cast<qps_ctx*>(c), [&] {
        need(c->have_geom, "build_geometry first");
        const int nI = int(c->geom.interfaces.size());
        if (I) *I = nI;
        if (n_nodes)
            for (int j = 0; j < nI; ++j) n_nodes[j] = c->geom.interfaces[j].quad.total();
        if (y_U) *y_U = c->geom.frame.y_U;
        if (y_D) *y_D = c->geom.frame.y_D;
        if (c->have_prob) {
            if (K) *K = c->prob.K;
            if (k)
                for (int i = 0; i <= nI; ++i) k[i] = c->prob.k[i];
            if (alpha) *alpha = {c->prob.alpha.real(), c->prob.alpha.imag()};
        } else if (K) {
            *K = 0;
        }
    });
}

int qps_interface_nodes(const qps_ctx* c, int j, double* nodes, double* normals, double* w, double* sp) {
    return guarded(const_cast<qps_ctx*>(c), [&] {
        need(c->have_geom && j >= 0 && j < int(c->geom.interfaces.size()), "bad interface");
        const auto& q = c->geom.interfaces[j].quad;
        for (int i = 0; i < q.total(); ++i) {
            if (nodes) { nodes[2 * i] = q.nodes[i].x; nodes[2 * i + 1] = q.nodes[i].y; }
            if (normals) { normals[2 * i] = q.normals[i].x; normals[2 * i + 1] = q.normals[i].y; }
            if (w) w[i] = q.weights[i];
            if (sp) sp[i] = q.speeds[i];
        }
    });
}

int qps_precompute_shift_blocks(qps_ctx* c) {
    return guarded(c, [&] {
        need(c->have_prob, "make_problem first");
        const auto t0 = clk::now();
        c->cache = precompute_shift_blocks(c->prob, c->num);
        c->fill_evals = c->cache->fill_evals;
        c->times.fill_ms = ms_since(t0);
    });
}

int qps_assemble_system(qps_ctx* c) {
    return guarded(c, [&] {
        need(c->cache.has_value(), "precompute_shift_blocks first");
        const auto t0 = clk::now();
        c->sys = assemble_system(c->prob, *c->cache, c->num);
        c->times.assemble_ms = ms_since(t0);
    });
}

int qps_schur_complement(qps_ctx* c) {
    return guarded(c, [&] {
        need(c->sys.has_value(), "assemble_system first");
        const auto t0 = clk::now();
        c->ps = schur_complement(*c->sys);
        c->times.schur_ms = ms_since(t0);
    });
}

int qps_block_lu_solve(qps_ctx* c) {
    return guarded(c, [&] {
        need(c->ps.has_value(), "schur_complement first");
        const auto t0 = clk::now();
        c->eta = block_lu_solve(*c->ps);
        c->times.solve_ms = ms_since(t0);
    });
}

int qps_block_lu_solve_blocks(qps_ctx* c, int I, int n, const qps_cplx* Ad, const qps_cplx* Au, const qps_cplx* Al,
                              const qps_cplx* f, qps_cplx* eta) {
    return guarded(c, [&] {
        PeriodizedSystem ps;
        ps.I = I;
        ps.P = 0;
        ps.K = 0;
        ps.N.assign(I, n / 2);
        const size_t nn = size_t(n) * n;
        auto mat = [&](const qps_cplx* p) {
            Mat m(n, n);
            std::memcpy(m.data(), p, sizeof(cd) * nn);
            return m;
        };
        for (int j = 0; j < I; ++j) ps.Ap_diag.push_back(mat(Ad + j * nn));
        for (int j = 0; j + 1 < I; ++j) {
            ps.Ap_super.push_back(mat(Au + j * nn));
            ps.Ap_sub.push_back(mat(Al + j * nn));
        }
        ps.f.resize(n);
        std::memcpy(ps.f.data(), f, sizeof(cd) * n);
        const auto e = block_lu_solve(ps);
        for (int j = 0; j < I; ++j) std::memcpy(eta + size_t(j) * n, e[j].data(), sizeof(cd) * n);
    });
}

int qps_recover_aux(qps_ctx* c) {
    return guarded(c, [&] {
        need(c->ps.has_value() && !c->eta.empty(), "block_lu_solve first");
        const auto t0 = clk::now();
        Solution s;
        recover_aux(*c->ps, c->eta, s);
        s.flux_error = flux_error(s, c->prob);
        c->sol = std::move(s);
        c->times.recover_ms = ms_since(t0);
    });
}

int qps_solve(qps_ctx* c) {
    const auto t0 = clk::now();
    int s = qps_precompute_shift_blocks(c);
    if (s == QPS_OK) s = qps_assemble_system(c);
    if (s == QPS_OK) s = qps_schur_complement(c);
    if (s == QPS_OK) s = qps_block_lu_solve(c);
    if (s == QPS_OK) s = qps_recover_aux(c);
    if (c) c->times.total_ms = ms_since(t0);
    return s;
}

int qps_get_solution(const qps_ctx* c, qps_cplx* eta, qps_cplx* cc, qps_cplx* aU, qps_cplx* aD, double* lsq,
                     double* max_lsq) {
    return guarded(const_cast<qps_ctx*>(c), [&] {
        need(c->sol.has_value(), "no solution");
        const Solution& s = *c->sol;
        if (eta) {
            size_t o = 0;
            for (const auto& e : s.eta) {
                std::memcpy(eta + o, e.data(), sizeof(cd) * e.size());
                o += e.size();
            }
        }
        if (cc) {
            size_t o = 0;
            for (const auto& v : s.c) {
                std::memcpy(cc + o, v.data(), sizeof(cd) * v.size());
                o += v.size();
            }
        }
        if (aU) std::memcpy(aU, s.aU.data(), sizeof(cd) * s.aU.size());
        if (aD) std::memcpy(aD, s.aD.data(), sizeof(cd) * s.aD.size());
        if (lsq)
            for (size_t i = 0; i < c->ps->lsq_residual.size(); ++i) lsq[i] = c->ps->lsq_residual[i];
        if (max_lsq) *max_lsq = s.max_lsq_residual;
    });
}

int qps_set_solution(qps_ctx* c, const qps_cplx* eta, const qps_cplx* cc, const qps_cplx* aU, const qps_cplx* aD) {
    return guarded(c, [&] {
        need(c->have_prob, "make_problem first");
        const int I = c->prob.n_interfaces(), P = c->num.P, nrb = 2 * c->prob.K + 1;
        Solution s;
        size_t o = 0;
        for (int j = 0; j < I; ++j) {
            const int n = 2 * c->geom.interfaces[j].quad.total();
            Vec e(n);
            for (int i = 0; i < n; ++i) e(i) = cd(eta[o + i].re, eta[o + i].im);
            s.eta.push_back(e);
            o += n;
        }
        for (int l = 0; l <= I; ++l) {
            Vec v(P);
            for (int i = 0; i < P; ++i) v(i) = cd(cc[size_t(l) * P + i].re, cc[size_t(l) * P + i].im);
            s.c.push_back(v);
        }
        s.aU = Vec(nrb);
        s.aD = Vec(nrb);
        for (int i = 0; i < nrb; ++i) {
            s.aU(i) = cd(aU[i].re, aU[i].im);
            s.aD(i) = cd(aD[i].re, aD[i].im);
        }
        s.flux_error = flux_error(s, c->prob);
        c->sol = s;
    });
}

// residual_suite / interface_matching_residual (postprocess.hpp:263-399)
int qps_residual_suite(qps_ctx* c, int n_interfaces, const int* interfaces, double* wall_qp, double* radiation,
                       double* interface_res) {
    return guarded(c, [&] {
        need(c->sol.has_value(), "no solution");
        const ResidualReport r = residual_suite(*c->sol, c->prob, c->num,
                                                std::vector<int>(interfaces, interfaces + n_interfaces));
        if (wall_qp) *wall_qp = r.wall_qp;
        if (radiation) *radiation = r.radiation;
        if (interface_res) *interface_res = r.interface;
    });
}

int qps_interface_matching_residual(qps_ctx* c, int j, int n_probe, double* out) {
    return guarded(c, [&] {
        need(c->sol.has_value(), "no solution");
        need(j >= 0 && j < c->prob.n_interfaces(), "interface_matching_residual: interface index out of range");
        need(n_probe >= 1, "interface_matching_residual: n_probe >= 1");
        const double r = interface_matching_residual(*c->sol, c->prob, c->num, j, n_probe);
        if (out) *out = r;
    });
}

int qps_reflection_transmission(const qps_ctx* c, double* R, double* T, double* fe, double* kappa, qps_cplx* kU,
                                qps_cplx* kD, int* pu, int* pd) {
    return guarded(const_cast<qps_ctx*>(c), [&] {
        need(c->sol.has_value(), "no solution");
        const SpectrumRow row = reflection_transmission(*c->sol, c->prob);
        if (R) *R = row.R;
        if (T) *T = row.T;
        if (fe) *fe = row.flux_error;
        for (size_t i = 0; i < row.up.size(); ++i) {
            if (kappa) kappa[i] = row.up[i].kappa;
            if (kU) kU[i] = {row.up[i].k_vert.real(), row.up[i].k_vert.imag()};
            if (kD) kD[i] = {row.down[i].k_vert.real(), row.down[i].k_vert.imag()};
            if (pu) pu[i] = row.up[i].propagating;
            if (pd) pd[i] = row.down[i].propagating;
        }
    });
}

// The reference has no sweep driver (proj/tests/test_sweep.cpp:1); this is the
// SPEC.md:505-547 composition of its building blocks.  mode 0: the cache is
// filled once; angles sharing alpha (|alpha_a - alpha_b| <= 1e-12) form a group
// whose interior elimination schur_interior (periodize.hpp:67-94) runs once,
// then per angle assemble_radiation / assemble_rhs / assemble_corners
// (assembly.hpp:407-460), schur_corners (periodize.hpp:98-121), block_lu_solve,
// recover_aux (tridiag.hpp:23-66).  mode 1: every angle independently
// (precompute_shift_blocks + assemble_system + solve_periodized).
int qps_sweep(qps_ctx* c, int n, const double* theta, int K, int mode, double* R, double* T, double* fe,
              qps_cplx* aU, qps_cplx* aD, int* status) {
    return guarded(c, [&] {
        need(c->have_prob, "make_problem first (sets omega)");
        need(K > 0, "sweep needs a fixed K > 0");
        need(mode == 0 || mode == 1, "sweep: mode is 0 (accelerated) or 1 (independent)");
        const double omega = c->prob.omega;
        const int nrb = 2 * K + 1;
        const auto t0 = clk::now();
        std::optional<ShiftBlockCache> cache;
        const double nan = std::nan("");
        c->sweep_group.assign(n, -1);
        c->sweep_ngroups = 0;
        c->sweep_interior = c->sweep_factorizations = 0;
        std::vector<std::optional<ScatteringProblem>> probs(n);
        for (int a = 0; a < n; ++a) {
            if (R) R[a] = nan;
            if (T) T[a] = nan;
            if (fe) fe[a] = nan;
            qps_ctx tmp;
            const int st = guarded(&tmp, [&] { probs[a] = make_problem(c->stack, c->geom, omega, theta[a], K); });
            if (status) status[a] = st;
        }
        // alpha groups in order of first appearance
        std::vector<std::vector<int>> groups;
        std::vector<cd> reps;
        for (int a = 0; a < n; ++a) {
            if (!probs[a]) continue;
            int gi = -1;
            for (size_t r = 0; r < reps.size() && mode == 0; ++r)
                if (std::abs(probs[a]->alpha - reps[r]) <= 1e-12) {
                    gi = int(r);
                    break;
                }
            if (gi < 0) {
                gi = int(groups.size());
                groups.emplace_back();
                reps.push_back(probs[a]->alpha);
            }
            groups[gi].push_back(a);
            c->sweep_group[a] = gi;
        }
        c->sweep_ngroups = int(groups.size());
        auto emit = [&](int a, const Solution& s) {
            const SpectrumRow row = reflection_transmission(s, *probs[a]);
            if (R) R[a] = row.R;
            if (T) T[a] = row.T;
            if (fe) fe[a] = row.flux_error;
            for (int i = 0; i < nrb; ++i) {
                if (aU) aU[size_t(a) * nrb + i] = {s.aU(i).real(), s.aU(i).imag()};
                if (aD) aD[size_t(a) * nrb + i] = {s.aD(i).real(), s.aD(i).imag()};
            }
        };
        for (const auto& g : groups) {
            if (mode != 0) {  // independent: the whole pipeline per angle
                qps_ctx tmp;
                const int st = guarded(&tmp, [&] {
                    cache = precompute_shift_blocks(*probs[g[0]], c->num);
                    c->fill_evals = cache->fill_evals;
                    const BlockSystem sys = assemble_system(*probs[g[0]], *cache, c->num);
                    ++c->sweep_interior;
                    ++c->sweep_factorizations;
                    emit(g[0], solve_periodized(sys));
                });
                if (status) status[g[0]] = st;
                continue;
            }
            qps_ctx tmp;
            std::optional<BlockSystem> sys;
            std::optional<InteriorSchur> interior;
            const int st = guarded(&tmp, [&] {
                if (!cache) {  // mode 0: the first valid angle fills the cache
                    cache = precompute_shift_blocks(*probs[g[0]], c->num);
                    c->fill_evals = cache->fill_evals;
                }
                sys = assemble_system(*probs[g[0]], *cache, c->num);
                interior = schur_interior(*sys);
                ++c->sweep_interior;
            });
            if (st != QPS_OK) {
                for (int a : g)
                    if (status) status[a] = st;
                continue;
            }
            for (int a : g) {
                const int sa = guarded(&tmp, [&] {
                    assemble_radiation(*probs[a], *cache, *sys);
                    assemble_rhs(*probs[a], *sys);
                    assemble_corners(*sys);
                    const PeriodizedSystem ps = schur_corners(*interior, *sys);
                    Solution s;
                    recover_aux(ps, block_lu_solve(ps), s);
                    ++c->sweep_factorizations;
                    emit(a, s);
                });
                if (status) status[a] = sa;
            }
        }
        c->times.fill_ms = ms_since(t0);
    });
}

int qps_sweep_info(const qps_ctx* c, int cap, int* alpha_group, int* n_groups, uint64_t* n_interior,
                   uint64_t* n_factorizations) {
    if (!c) return QPS_ERR_USAGE;
    for (int a = 0; alpha_group && a < cap && a < int(c->sweep_group.size()); ++a) alpha_group[a] = c->sweep_group[a];
    if (n_groups) *n_groups = c->sweep_ngroups;
    if (n_interior) *n_interior = c->sweep_interior;
    if (n_factorizations) *n_factorizations = c->sweep_factorizations;
    return QPS_OK;
}

// plan_sweep: angles uniform in kappa_0 = k_1 cos(theta) with
// spacing 2 pi / (n d) inside (theta_lo, theta_hi), so alpha takes n values
int qps_plan_sweep(qps_ctx* c, int n_alpha, double theta_lo, double theta_hi, int cap, double* theta,
                   int* alpha_group, int* n_angles) {
    return guarded(c, [&] {
        need(c->have_prob, "make_problem first (sets k_1)");
        if (n_alpha < 1) throw ConfigError("plan_sweep: n >= 1 alpha values required");
        if (!(theta_lo > -pi && theta_hi < 0.0 && theta_lo < theta_hi))
            throw ConfigError("plan_sweep: theta range must satisfy -pi < lo < hi < 0");
        const double k1 = c->prob.k.front(), d = c->stack.d;
        const double klo = k1 * std::cos(theta_lo), khi = k1 * std::cos(theta_hi), dk = 2.0 * pi / (n_alpha * d);
        int cnt = 0;
        for (int j = 0;; ++j) {
            const double kap = klo + (j + 0.5) * dk;
            if (kap >= khi) break;
            if (cnt < cap) {
                if (theta) theta[cnt] = -std::acos(kap / k1);
                if (alpha_group) alpha_group[cnt] = j % n_alpha;
            }
            ++cnt;
        }
        if (n_angles) *n_angles = cnt;
    });
}

int qps_evaluate_field(qps_ctx* c, int n, const double* xy, qps_cplx* u_scat, qps_cplx* u_tot, int* region,
                       int* layer) {
    return guarded(c, [&] {
        need(c->sol.has_value(), "no solution (solve first)");
        std::vector<Vec2> pts(n);
        for (int i = 0; i < n; ++i) pts[i] = Vec2{xy[2 * i], xy[2 * i + 1]};
        const std::vector<FieldSample> fs = evaluate_field(*c->sol, c->prob, pts);
        for (int i = 0; i < n; ++i) {
            if (u_scat) u_scat[i] = {fs[i].u_scattered.real(), fs[i].u_scattered.imag()};
            if (u_tot) u_tot[i] = {fs[i].u_total.real(), fs[i].u_total.imag()};
            if (region) region[i] = fs[i].region == Region::AboveU ? 0 : fs[i].region == Region::Layer ? 1 : 2;
            if (layer) layer[i] = fs[i].layer;
        }
    });
}

int qps_download_block(const qps_ctx* c, int kind, int i, qps_cplx* out, int* rows, int* cols) {
    return guarded(const_cast<qps_ctx*>(c), [&] {
        if (kind < 32) {
            need(c->sys.has_value(), "assemble_system first");
            const BlockSystem& s = *c->sys;
            switch (kind) {
                case QPS_BLK_A_DIAG: return put(pick(s.A_diag, i), out, rows, cols);
                case QPS_BLK_A_SUPER: return put(pick(s.A_super, i), out, rows, cols);
                case QPS_BLK_A_SUB: return put(pick(s.A_sub, i), out, rows, cols);
                case QPS_BLK_B_SELF: return put(pick(s.B_self, i), out, rows, cols);
                case QPS_BLK_B_BELOW: return put(pick(s.B_below, i), out, rows, cols);
                case QPS_BLK_C_SELF: return put(pick(s.C_self, i), out, rows, cols);
                case QPS_BLK_C_ABOVE: return put(pick(s.C_above, i), out, rows, cols);
                case QPS_BLK_Q: return put(pick(s.Q, i), out, rows, cols);
                case QPS_BLK_Z_U: return put(s.Z_U, out, rows, cols);
                case QPS_BLK_Z_D: return put(s.Z_D, out, rows, cols);
                case QPS_BLK_V_U: return put(s.V_U, out, rows, cols);
                case QPS_BLK_V_D: return put(s.V_D, out, rows, cols);
                case QPS_BLK_W_U: return put(s.W_U, out, rows, cols);
                case QPS_BLK_W_D: return put(s.W_D, out, rows, cols);
                case QPS_BLK_F: return put(Mat(s.f), out, rows, cols);
                case QPS_BLK_BP_FIRST: return put(s.Bp_first, out, rows, cols);
                case QPS_BLK_BP_LAST: return put(s.Bp_last, out, rows, cols);
                case QPS_BLK_CP_FIRST: return put(s.Cp_first, out, rows, cols);
                case QPS_BLK_CP_LAST: return put(s.Cp_last, out, rows, cols);
                case QPS_BLK_QP_FIRST: return put(s.Qp_first, out, rows, cols);
                case QPS_BLK_QP_LAST: return put(s.Qp_last, out, rows, cols);
                default: throw UsageError("qps oracle: unknown block kind");
            }
        }
        need(c->ps.has_value(), "schur_complement first");
        const PeriodizedSystem& p = *c->ps;
        switch (kind) {
            case QPS_BLK_AP_DIAG: return put(pick(p.Ap_diag, i), out, rows, cols);
            case QPS_BLK_AP_SUPER: return put(pick(p.Ap_super, i), out, rows, cols);
            case QPS_BLK_AP_SUB: return put(pick(p.Ap_sub, i), out, rows, cols);
            case QPS_BLK_X_FIRST: return put(p.X_first, out, rows, cols);
            case QPS_BLK_X_ABOVE: return put(pick(p.X_above, i), out, rows, cols);
            case QPS_BLK_X_SELF: return put(pick(p.X_self, i), out, rows, cols);
            case QPS_BLK_X_LAST: return put(p.X_last, out, rows, cols);
            default: throw UsageError("qps oracle: unknown block kind");
        }
    });
}

int qps_fill_evals(const qps_ctx* c, uint64_t* reference, uint64_t* performed) {
    if (!c) return QPS_ERR_USAGE;
    if (reference) *reference = c->fill_evals;
    if (performed) *performed = c->fill_evals;
    return QPS_OK;
}

int qps_get_phase_times(const qps_ctx* c, qps_phase_times* t) {
    if (!c || !t) return QPS_ERR_USAGE;
    *t = c->times;
    return QPS_OK;
}

int qps_solver_diagnostics(const qps_ctx* c, qps_solver_diag* d) {
    if (!c || !d) return QPS_ERR_USAGE;
    *d = qps_solver_diag{-1, 0, 0.0, 0, 0.0, 0.0, 0, 0};  // the reference's block Thomas (tridiag.hpp:23-46)
    return QPS_OK;
}

int qps_hankel01(qps_ctx* c, int n, const double* x, qps_cplx* h0, qps_cplx* h1) {
    return guarded(c, [&] {
        for (int i = 0; i < n; ++i) {
            const HankelPair h = hankel01(x[i]);
            h0[i] = {h.h0.real(), h.h0.imag()};
            h1[i] = {h.h1.real(), h.h1.imag()};
        }
    });
}

int qps_qsolve(qps_ctx* c, int m, int p, int n, const qps_cplx* Q, const qps_cplx* R, qps_cplx* X, int* rank) {
    return guarded(c, [&] {
        Mat q(m, p), r(m, n);
        std::memcpy(q.data(), Q, sizeof(cd) * size_t(m) * p);
        std::memcpy(r.data(), R, sizeof(cd) * size_t(m) * n);
        const Mat x = qsolve(q, r);
        std::memcpy(X, x.data(), sizeof(cd) * size_t(p) * n);
        if (rank) {
            Eigen::CompleteOrthogonalDecomposition<Mat> cod;
            cod.setThreshold(qsolve_threshold());
            cod.compute(q);
            *rank = int(cod.rank());
        }
    });
}

int qps_debug_zgemm(qps_ctx* c, int M, int N, int K, const qps_cplx* A, const qps_cplx* B, qps_cplx* Cm) {
    return guarded(c, [&] {
        Mat a(M, K), b(K, N);
        std::memcpy(a.data(), A, sizeof(cd) * size_t(M) * K);
        std::memcpy(b.data(), B, sizeof(cd) * size_t(K) * N);
        const Mat r = a * b;
        std::memcpy(Cm, r.data(), sizeof(cd) * size_t(M) * N);
    });
}

int qps_prof_enable(qps_ctx* c, int) { return c ? QPS_OK : QPS_ERR_USAGE; }
int qps_prof_reset(qps_ctx* c) { return c ? QPS_OK : QPS_ERR_USAGE; }
int qps_prof_stats(qps_ctx*, int, char*, uint64_t*, double*, double*, double*, double*) { return 0; }
uint64_t qps_launch_count(void) { return 0; }
int qps_transfer_bytes(const qps_ctx* c, uint64_t* a, uint64_t* b) {
    if (!c) return QPS_ERR_USAGE;
    if (a) *a = 0;
    if (b) *b = 0;
    return QPS_OK;
}

int qps_measure_fp64_peaks(qps_ctx* c, double* a, double* b) {
    if (!c) return QPS_ERR_USAGE;
    if (a) *a = 0.0;
    if (b) *b = 0.0;
    return QPS_OK;
}

}  // extern "C"
