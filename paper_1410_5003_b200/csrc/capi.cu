// C-ABI of the B200 implementation (include/qpscat_b200.h).  Every entry point
// converts exceptions into qps_status codes following the reference's error
// taxonomy (errors.hpp:9-40) and never falls back to a CPU path.
#include <chrono>
#include <cstring>

#include "ctx.h"
#include "prof.h"

using namespace qpsb;

struct qps_ctx {
    Ctx c;
};

namespace {

template <class F>
int guarded(qps_ctx* h, F&& f) {
    if (!h) return QPS_ERR_USAGE;
    Ctx& c = h->c;
    c.err_msg.clear();
    c.err_layer = 0;
    c.err_bytes = 0;
    try {
        if (!c.host_only) QPS_CUDA(cudaSetDevice(c.device));
        f(c);
        return QPS_OK;
    } catch (const Error& e) {
        c.err_msg = e.what();
        c.err_layer = e.layer;
        c.err_bytes = e.bytes;
        return e.status;
    } catch (const std::exception& e) {
        c.err_msg = e.what();
        return QPS_ERR_INTERNAL;
    }
}

void need(bool ok, const char* what) {
    if (!ok) fail(QPS_ERR_USAGE, std::string("qpscat_b200: ") + what);
}

void need_device(const Ctx& c) {
    if (c.host_only) fail(QPS_ERR_CUDA, "qpscat_b200: host-only context (device -1) cannot run device work");
}

void prepare(Ctx& c, bool check_solvable = true) {
    need(c.have_prob, "make_problem first");
    setup_dims(c, check_solvable);
}

void get_block(const Ctx& c, const cplx* base, int ld, int rows, int cols, qps_cplx* out, int* r, int* cc) {
    if (r) *r = rows;
    if (cc) *cc = cols;
    if (!out || rows == 0 || cols == 0) return;
    QPS_CUDA(cudaMemcpy2DAsync(out, sizeof(cplx) * rows, base, sizeof(cplx) * ld, sizeof(cplx) * rows, cols,
                               cudaMemcpyDeviceToHost, c.stream));
    QPS_CUDA(cudaStreamSynchronize(c.stream));
}

void zero_block(int* r, int* cc) {
    if (r) *r = 0;
    if (cc) *cc = 0;
}

void set_spec(StackDesc& st, int n, const qps_interface_spec* ifs) {
    st.cosc.resize(n);
    st.sinc.resize(n);
    st.verts.resize(n);
    st.nodes.resize(n);
    st.ifaces.resize(n);
    for (int j = 0; j < n; ++j) {
        const auto& s = ifs[j];
        st.cosc[j].assign(s.cosc, s.cosc + (s.cosc ? s.n_cos : 0));
        st.sinc[j].assign(s.sinc, s.sinc + (s.sinc ? s.n_sin : 0));
        st.verts[j].assign(s.vertices, s.vertices + (s.vertices ? 2 * s.n_vertices : 0));
        st.nodes[j].assign(s.nodes, s.nodes + (s.nodes ? s.n_nodes : 0));
        qps_interface_spec t = s;
        t.cosc = st.cosc[j].data();
        t.sinc = st.sinc[j].data();
        t.vertices = st.verts[j].data();
        t.nodes = st.nodes[j].data();
        t.n_cos = int(st.cosc[j].size());
        t.n_sin = int(st.sinc[j].size());
        t.n_vertices = int(st.verts[j].size() / 2);
        t.n_nodes = int(st.nodes[j].size());
        st.ifaces[j] = t;
    }
}

void run_fill(Ctx& c) {
    Timer t(c, &c.times.fill_ms);
    fill_system_fused(c);
}

}  // namespace

extern "C" {

int qps_abi_version(void) { return QPS_ABI_VERSION; }
const char* qps_backend_name(void) { return "b200-cuda"; }

qps_ctx* qps_create(int device) {
    if (device == -1) {  // host-only context for CPU-side logic (tests, planning)
        auto* h = new qps_ctx();
        h->c.host_only = true;
        h->c.device = -1;
        return h;
    }
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0 || device < 0 || device >= n) return nullptr;
    auto* h = new qps_ctx();
    h->c.device = device;
    try {
        QPS_CUDA(cudaSetDevice(device));
        // the latency-bound chains get the higher priorities (the corner least
        // squares, a few CTAs, above the main stream); the throughput-bound side
        // GEMMs (side2: the low-rank sample) fill the SMs the chains leave idle
        // instead of starving them
        int prio_lo = 0, prio_hi = 0;
        QPS_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        const int prio_main = prio_hi < prio_lo ? prio_hi + 1 : prio_hi;
        QPS_CUDA(cudaStreamCreateWithPriority(&h->c.stream, cudaStreamNonBlocking, prio_main));
        QPS_CUDA(cudaStreamCreateWithPriority(&h->c.side, cudaStreamNonBlocking, prio_hi));
        const char* sp = getenv("QPS_SAMPLE_PRIO");  // A/B: "main" puts side2 level with the main stream
        QPS_CUDA(cudaStreamCreateWithPriority(&h->c.side2, cudaStreamNonBlocking,
                                              (sp && !strcmp(sp, "main")) ? prio_main
                                              : (sp && !strcmp(sp, "hi")) ? prio_hi : prio_lo));
        QPS_CUDA(cudaStreamCreateWithPriority(&h->c.side3, cudaStreamNonBlocking, prio_lo));
        QPS_CUDA(cudaEventCreateWithFlags(&h->c.ev_fork, cudaEventDisableTiming));
        QPS_CUDA(cudaEventCreateWithFlags(&h->c.ev_fill, cudaEventDisableTiming));
        QPS_CUDA(cudaEventCreateWithFlags(&h->c.ev_sample, cudaEventDisableTiming));
        QPS_CUDA(cudaEventCreateWithFlags(&h->c.ev_anorm, cudaEventDisableTiming));
        QPS_CUDA(cudaEventCreateWithFlags(&h->c.ev_factor, cudaEventDisableTiming));
        QPS_CUDA(cudaEventCreateWithFlags(&h->c.ev_l0, cudaEventDisableTiming));
        QPS_CUDA(cudaEventCreate(&h->c.ev0));
        QPS_CUDA(cudaEventCreate(&h->c.ev1));
        upload_hankel_tables();
    } catch (...) {
        delete h;
        return nullptr;
    }
    return h;
}

void qps_destroy(qps_ctx* h) {
    if (!h) return;
    if (h->c.host_only) {
        delete h;
        return;
    }
    cudaSetDevice(h->c.device);
    cudaStreamSynchronize(h->c.stream);
    if (h->c.ev0) cudaEventDestroy(h->c.ev0);
    if (h->c.ev1) cudaEventDestroy(h->c.ev1);
    cudaStream_t s = h->c.stream, s2 = h->c.side, s3 = h->c.side2, s4 = h->c.side3;
    if (s2) cudaStreamSynchronize(s2);
    if (s3) cudaStreamSynchronize(s3);
    if (s4) cudaStreamSynchronize(s4);
    for (cudaEvent_t e : {h->c.ev_fork, h->c.ev_fill, h->c.ev_sample, h->c.ev_anorm, h->c.ev_factor, h->c.ev_l0, h->c.ev_f0,
                          h->c.ev_f1, h->c.ev_geo, h->c.ev_fillB, h->c.ev_rhs, h->c.ev_rank})
        if (e) cudaEventDestroy(e);
    std::vector<cudaStream_t> l0s;
    if (h->c.lsq_stream) {
        cudaStreamSynchronize(h->c.lsq_stream);
        l0s.push_back(h->c.lsq_stream);
    }
    for (int i = 0; i < qpsb::Ctx::kL0MaxChunks; ++i) {
        if (h->c.l0_s[i]) {
            cudaStreamSynchronize(h->c.l0_s[i]);
            l0s.push_back(h->c.l0_s[i]);
        }
        if (h->c.l0_ev[i]) cudaEventDestroy(h->c.l0_ev[i]);
    }
    delete h;
    for (cudaStream_t x : l0s) cudaStreamDestroy(x);
    if (s) cudaStreamDestroy(s);
    if (s2) cudaStreamDestroy(s2);
    if (s3) cudaStreamDestroy(s3);
    if (s4) cudaStreamDestroy(s4);
}

int qps_last_error(const qps_ctx* h, char* msg, size_t cap, int* layer, uint64_t* bytes) {
    if (!h) return QPS_ERR_USAGE;
    if (msg && cap) {
        std::strncpy(msg, h->c.err_msg.c_str(), cap - 1);
        msg[cap - 1] = 0;
    }
    if (layer) *layer = h->c.err_layer;
    if (bytes) *bytes = h->c.err_bytes;
    return QPS_OK;
}

int qps_set_num_threads(qps_ctx* h, int) { return h ? QPS_OK : QPS_ERR_USAGE; }

int qps_set_qsolve_threshold(qps_ctx* h, double th) {
    return guarded(h, [&](Ctx& c) { c.qsolve_th0 = th; });
}

int qps_set_refine(qps_ctx* h, int steps) {
    return guarded(h, [&](Ctx& c) {
        need(steps >= -1 && steps <= 4, "refine: steps in [-1, 4]");
        c.refine = steps;
    });
}

int qps_build_geometry(qps_ctx* h, double d, int n_layers, const double* eps, const double* mu, int n_ifaces,
                       const qps_interface_spec* ifs, const qps_numerics* num) {
    return guarded(h, [&](Ctx& c) {
        need(num != nullptr && eps != nullptr, "numerics and epsilon required");
        c.have_geom = c.have_prob = false;
        c.cache_valid = false;
        c.sys_valid = c.ps_valid = c.eta_valid = c.have_sol = false;
        StackDesc st;
        st.d = d;
        for (int i = 0; i < n_layers; ++i) {
            st.eps.push_back(eps[i]);
            st.mu.push_back(mu ? mu[i] : 1.0);
        }
        set_spec(st, n_ifaces, ifs);
        Numerics nm;
        nm.P = num->P;
        nm.Mw = num->Mw;
        nm.M = num->M;
        nm.K = num->K;
        nm.R = num->R;
        nm.grading_q = num->grading_q;
        nm.clearance = num->clearance;
        nm.memory_budget = num->memory_budget;
        c.stack = std::move(st);
        c.num = nm;
        static const bool htrace = getenv("QPS_HOST_TRACE") != nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        c.geo = build_geometry(c.stack, c.num);
        const auto t1 = std::chrono::steady_clock::now();
        if (!c.host_only) upload_geometry(c);
        const auto t2 = std::chrono::steady_clock::now();
        if (htrace)
            fprintf(stderr, "qps_build_geometry: build %.3f ms, upload %.3f ms\n",
                    std::chrono::duration<double, std::milli>(t1 - t0).count(),
                    std::chrono::duration<double, std::milli>(t2 - t1).count());
        c.have_geom = true;
    });
}

int qps_make_problem(qps_ctx* h, double omega, double theta, int K) {
    return guarded(h, [&](Ctx& c) {
        need(c.have_geom, "build_geometry first");
        c.prob = make_problem(c.stack, c.geo, omega, theta, K);
        c.have_prob = true;
        if (c.cache_valid && c.cache_k != c.prob.k) c.cache_valid = false;  // the cache depends on omega only
        c.sys_valid = c.ps_valid = c.eta_valid = c.have_sol = false;
    });
}

int qps_problem_info(const qps_ctx* h, int* I, int* K, int* n_nodes, double* k, qps_cplx* alpha, double* y_U,
                     double* y_D) {
    return guarded(const_cast<qps_ctx*>(h), [&](Ctx& c) {
        need(c.have_geom, "build_geometry first");
        if (I) *I = c.geo.I;
        if (n_nodes)
            for (int j = 0; j < c.geo.I; ++j) n_nodes[j] = c.geo.ifaces[j].N();
        if (y_U) *y_U = c.geo.y_U;
        if (y_D) *y_D = c.geo.y_D;
        if (c.have_prob) {
            if (K) *K = c.prob.K;
            if (k)
                for (size_t i = 0; i < c.prob.k.size(); ++i) k[i] = c.prob.k[i];
            if (alpha) *alpha = qps_cplx{c.prob.ar, c.prob.ai};
        } else if (K) {
            *K = 0;
        }
    });
}

int qps_interface_nodes(const qps_ctx* h, int j, double* nodes, double* normals, double* w, double* sp) {
    return guarded(const_cast<qps_ctx*>(h), [&](Ctx& c) {
        need(c.have_geom && j >= 0 && j < c.geo.I, "bad interface");
        const auto& q = c.geo.ifaces[j];
        for (int i = 0; i < q.N(); ++i) {
            if (nodes) { nodes[2 * i] = q.x[i]; nodes[2 * i + 1] = q.y[i]; }
            if (normals) { normals[2 * i] = q.nx[i]; normals[2 * i + 1] = q.ny[i]; }
            if (w) w[i] = q.w[i];
            if (sp) sp[i] = q.speed[i];
        }
    });
}

int qps_precompute_shift_blocks(qps_ctx* h) {
    return guarded(h, [&](Ctx& c) {
        prepare(c, false);  // memory budget guard, assembly.hpp:216-223
        c.sys_valid = c.ps_valid = c.eta_valid = c.have_sol = false;
        if (c.host_only) {
            c.ref_evals = reference_fill_evals(c.geo);
            return;
        }
        Timer t(c, &c.times.fill_ms);
        cache_fill(c);
    });
}

int qps_assemble_system(qps_ctx* h) {
    return guarded(h, [&](Ctx& c) {
        need_device(c);
        prepare(c);
        if (!(c.cache_valid && c.cache_k == c.prob.k)) {
            Timer t(c, &c.times.fill_ms);
            cache_fill(c);
        }
        {
            Timer t(c, &c.times.assemble_ms);
            assemble_from_cache(c, {c.prob});
        }
        c.ps_separate = true;
    });
}

int qps_schur_complement(qps_ctx* h) {
    return guarded(h, [&](Ctx& c) {
        need_device(c);
        need(c.sys_valid, "assemble_system first");
        Timer t(c, &c.times.schur_ms);
        const Dims& D = c.dims;
        const size_t nb2 = size_t(D.nb) * D.nb;
        c.Apdiag.ensure(D.I * nb2);
        c.Apsup.ensure(std::max(1, D.I - 1) * nb2);
        c.Apsub.ensure(std::max(1, D.I - 1) * nb2);
        QPS_CUDA(cudaMemcpyAsync(c.Apdiag.p, c.Adiag.p, sizeof(cplx) * D.I * nb2, cudaMemcpyDeviceToDevice, c.stream));
        if (D.I > 1) {
            QPS_CUDA(cudaMemcpyAsync(c.Apsup.p, c.Asup.p, sizeof(cplx) * (D.I - 1) * nb2, cudaMemcpyDeviceToDevice,
                                     c.stream));
            QPS_CUDA(cudaMemcpyAsync(c.Apsub.p, c.Asub.p, sizeof(cplx) * (D.I - 1) * nb2, cudaMemcpyDeviceToDevice,
                                     c.stream));
        }
        schur(c, c.Apdiag.p, c.Apsup.p, c.Apsub.p);
        c.ps_separate = true;
    });
}

int qps_block_lu_solve(qps_ctx* h) {
    return guarded(h, [&](Ctx& c) {
        need_device(c);
        need(c.ps_valid, "schur_complement first");
        Timer t(c, &c.times.solve_ms);
        if (c.ps_separate) bcr_solve(c, c.Apdiag.p, c.Apsup.p, c.Apsub.p);
        else bcr_solve(c, c.Adiag.p, c.Asup.p, c.Asub.p);
        c.ps_valid = false;  // factors overwrite A'
    });
}

int qps_block_lu_solve_blocks(qps_ctx* h, int I, int n, const qps_cplx* Ad, const qps_cplx* Au, const qps_cplx* Al,
                              const qps_cplx* f, qps_cplx* eta) {
    return guarded(h, [&](Ctx& c) {
        need(I >= 1 && n >= 1, "block_lu_solve_blocks: empty system");
        need_device(c);
        const size_t nn = size_t(n) * n;
        Dims D;
        D.I = I;
        D.nb = n;
        D.N.assign(I, n / 2);
        c.dims = D;
        DBuf<cplx> dA, dU, dL;
        dA.ensure(I * nn);
        dU.ensure(std::max(1, I - 1) * nn);
        dL.ensure(std::max(1, I - 1) * nn);
        c.f.ensure(n);
        QPS_CUDA(cudaMemcpyAsync(dA.p, Ad, sizeof(cplx) * I * nn, cudaMemcpyHostToDevice, c.stream));
        if (I > 1) {
            QPS_CUDA(cudaMemcpyAsync(dU.p, Au, sizeof(cplx) * (I - 1) * nn, cudaMemcpyHostToDevice, c.stream));
            QPS_CUDA(cudaMemcpyAsync(dL.p, Al, sizeof(cplx) * (I - 1) * nn, cudaMemcpyHostToDevice, c.stream));
        }
        QPS_CUDA(cudaMemcpyAsync(c.f.p, f, sizeof(cplx) * n, cudaMemcpyHostToDevice, c.stream));
        {
            Timer t(c, &c.times.solve_ms);
            bcr_solve(c, dA.p, dU.p, dL.p);
        }
        QPS_CUDA(cudaMemcpyAsync(eta, c.F.p, sizeof(cplx) * I * size_t(n), cudaMemcpyDeviceToHost, c.stream));
        QPS_CUDA(cudaStreamSynchronize(c.stream));
        c.sys_valid = c.ps_valid = c.eta_valid = c.have_sol = false;
    });
}

int qps_recover_aux(qps_ctx* h) {
    return guarded(h, [&](Ctx& c) {
        need_device(c);
        need(c.eta_valid, "block_lu_solve first");
        Timer t(c, &c.times.recover_ms);
        recover(c);
    });
}

int qps_solve(qps_ctx* h) {
    return guarded(h, [&](Ctx& c) {
        prepare(c);  // input validation first (same errors with or without a device)
        need_device(c);
        cudaEvent_t t0, t1;
        QPS_CUDA(cudaEventCreate(&t0));
        QPS_CUDA(cudaEventCreate(&t1));
        QPS_CUDA(cudaEventRecord(t0, c.stream));
        struct Total {
            Ctx& c;
            cudaEvent_t a, b;
            ~Total() {
                cudaEventRecord(b, c.stream);
                cudaEventSynchronize(b);
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                c.times.total_ms = ms;
                cudaEventDestroy(a);
                cudaEventDestroy(b);
            }
        } total{c, t0, t1};
        c.ps_separate = false;
        c.times.factor_ms = 0.0;
        tl_mark(c, "start", c.stream);
        for (int attempt = 0;; ++attempt) {
            c.fill_overlap = true;  // the Schur least squares start while the big blocks fill
            c.sketch_in_fill = true;
            c.sketch_launched = false;
            try {
                run_fill(c);
            } catch (...) {
                c.fill_overlap = c.sketch_in_fill = false;
                throw;
            }
            c.fill_overlap = c.sketch_in_fill = false;
            tl_mark(c, "fill", c.stream);
            c.times.assemble_ms = 0.0;
            if (!c.sketch_launched) lr_sample_async(c);  // overlaps the Schur least squares
            {
                Timer t(c, &c.times.schur_ms);
                static const bool no_defer = [] {  // QPS_DEFER=0: form the coupling updates explicitly (A/B)
                    const char* e = getenv("QPS_DEFER");
                    return e && !strcmp(e, "0");
                }();
                schur(c, c.Adiag.p, c.Asup.p, c.Asub.p, !no_defer, true);
            }
            tl_mark(c, "schur", c.stream);
            c.sys_valid = false;  // A now holds A'
            try {
                Timer t(c, &c.times.solve_ms);
                c.allow_early = true;
                bcr_solve(c, c.Adiag.p, c.Asup.p, c.Asub.p);
                c.allow_early = false;
            } catch (const Error& e) {
                c.allow_early = false;
                // couplings not low rank (or not at the truncated width) after the
                // early level-0 factorization: once more, dense (full width)
                if (solve_retry(c, e)) continue;
                c.force_dense = c.lr_full_width = false;
                throw;
            }
            c.force_dense = c.lr_full_width = false;
            break;
        }
        c.ps_valid = false;
        {
            Timer t(c, &c.times.recover_ms);
            recover(c);
        }
        schur_finish(c);  // the per-layer LSQ residuals (low-priority stream)
        tl_mark(c, "recover", c.stream);
        tl_report(c);
    });
}

int qps_get_solution(const qps_ctx* h, qps_cplx* eta, qps_cplx* cc, qps_cplx* aU, qps_cplx* aD, double* lsq,
                     double* max_lsq) {
    return guarded(const_cast<qps_ctx*>(h), [&](Ctx& c) {
        need(c.have_sol, "no solution");
        if (eta) std::memcpy(eta, c.h_eta.p, sizeof(cplx) * c.h_eta_n);
        if (cc) std::memcpy(cc, c.h_c.data(), sizeof(cplx) * c.h_c.size());
        if (aU) std::memcpy(aU, c.h_aU.data(), sizeof(cplx) * c.h_aU.size());
        if (aD) std::memcpy(aD, c.h_aD.data(), sizeof(cplx) * c.h_aD.size());
        if (lsq)
            for (size_t i = 0; i < c.lsq.size(); ++i) lsq[i] = c.lsq[i];
        if (max_lsq) *max_lsq = c.max_lsq;
    });
}

int qps_set_solution(qps_ctx* h, const qps_cplx* eta, const qps_cplx* cc, const qps_cplx* aU, const qps_cplx* aD) {
    return guarded(h, [&](Ctx& c) {
        need_device(c);
        need(c.have_prob, "make_problem first");
        need(eta && cc && aU && aD, "set_solution: null array");
        if (c.dims.nb == 0 || c.dims.I != c.geo.I || c.dims.K != c.prob.K) setup_dims(c, false);
        c.dims.nsys = 1;
        const Dims& D = c.dims;
        const int I = D.I, nrb = 2 * c.prob.K + 1;
        size_t neta = 0;
        for (int j = 0; j < I; ++j) neta += 2 * size_t(D.N[j]);
        c.h_eta.ensure(neta);
        c.h_eta_n = neta;
        std::memcpy(c.h_eta.p, eta, sizeof(cplx) * neta);
        c.F.ensure(size_t(I) * D.nb);
        c.F.zero(c.stream);
        size_t o = 0;
        for (int j = 0; j < I; ++j) {
            QPS_CUDA(cudaMemcpyAsync(c.F.p + size_t(j) * D.nb, eta + o, sizeof(cplx) * 2 * D.N[j],
                                     cudaMemcpyHostToDevice, c.stream));
            o += 2 * size_t(D.N[j]);
        }
        QPS_CUDA(cudaStreamSynchronize(c.stream));
        c.h_c.assign(reinterpret_cast<const cplx*>(cc), reinterpret_cast<const cplx*>(cc) + size_t(I + 1) * D.P);
        c.h_aU.assign(reinterpret_cast<const cplx*>(aU), reinterpret_cast<const cplx*>(aU) + nrb);
        c.h_aD.assign(reinterpret_cast<const cplx*>(aD), reinterpret_cast<const cplx*>(aD) + nrb);
        c.lsq.assign(I + 1, 0.0);
        c.max_lsq = 0.0;
        c.have_sol = true;
        c.eta_valid = true;
    });
}

int qps_residual_suite(qps_ctx* h, int n_interfaces, const int* interfaces, double* wall_qp, double* radiation,
                       double* interface_res) {
    return guarded(h, [&](Ctx& c) {
        need_device(c);
        need(c.have_sol, "no solution");
        need(n_interfaces >= 0 && (n_interfaces == 0 || interfaces), "residual_suite: bad interface list");
        residual_suite(c, std::vector<int>(interfaces, interfaces + n_interfaces), wall_qp, radiation, interface_res);
    });
}

int qps_interface_matching_residual(qps_ctx* h, int j, int n_probe, double* out) {
    return guarded(h, [&](Ctx& c) {
        need_device(c);
        need(c.have_sol, "no solution");
        const double r = interface_matching_residual(c, j, n_probe);
        if (out) *out = r;
    });
}

int qps_reflection_transmission(const qps_ctx* h, double* R, double* T, double* fe, double* kappa, qps_cplx* kU,
                                qps_cplx* kD, int* pu, int* pd) {
    return guarded(const_cast<qps_ctx*>(h), [&](Ctx& c) {
        need(c.have_sol, "no solution");
        host_spectrum(c, R, T, fe, kappa, reinterpret_cast<cplx*>(kU), reinterpret_cast<cplx*>(kD), pu, pd);
    });
}

int qps_sweep(qps_ctx* h, int n, const double* theta, int K, int mode, double* R, double* T, double* fe,
              qps_cplx* aU, qps_cplx* aD, int* status) {
    return guarded(h, [&](Ctx& c) {
        need_device(c);
        need(c.have_prob, "make_problem first (sets omega)");
        need(K > 0, "sweep needs a fixed K > 0");
        need(n >= 0 && (n == 0 || theta != nullptr), "sweep: bad angle list");
        need(mode == 0 || mode == 1, "sweep: mode is 0 (accelerated) or 1 (independent)");
        run_sweep(c, n, theta, K, mode, R, T, fe, reinterpret_cast<cplx*>(aU), reinterpret_cast<cplx*>(aD), status);
    });
}

int qps_plan_sweep(qps_ctx* h, int n_alpha, double theta_lo, double theta_hi, int cap, double* theta,
                   int* alpha_group, int* n_angles) {
    return guarded(h, [&](Ctx& c) {
        need(c.have_prob, "make_problem first (sets k_1)");
        const std::vector<double> th = plan_sweep_angles(c.prob.k.front(), c.geo.d, n_alpha, theta_lo, theta_hi);
        for (int j = 0; j < int(th.size()) && j < cap; ++j) {
            if (theta) theta[j] = th[j];
            if (alpha_group) alpha_group[j] = j % n_alpha;
        }
        if (n_angles) *n_angles = int(th.size());
    });
}

int qps_sweep_info(const qps_ctx* h, int cap, int* alpha_group, int* n_groups, uint64_t* n_interior,
                   uint64_t* n_factorizations) {
    if (!h) return QPS_ERR_USAGE;
    const Ctx& c = h->c;
    for (int a = 0; alpha_group && a < cap && a < int(c.sweep_group.size()); ++a) alpha_group[a] = c.sweep_group[a];
    if (n_groups) *n_groups = c.sweep_ngroups;
    if (n_interior) *n_interior = c.sweep_interior;
    if (n_factorizations) *n_factorizations = c.sweep_factorizations;
    return QPS_OK;
}

int qps_evaluate_field(qps_ctx* h, int n, const double* xy, qps_cplx* u_scat, qps_cplx* u_tot, int* region,
                       int* layer) {
    return guarded(h, [&](Ctx& c) {
        need_device(c);
        need(c.have_sol, "no solution (solve first)");
        need(n >= 0 && (n == 0 || xy != nullptr), "evaluate_field: bad point list");
        evaluate_field(c, n, xy, reinterpret_cast<cplx*>(u_scat), reinterpret_cast<cplx*>(u_tot), region, layer);
    });
}

int qps_download_block(const qps_ctx* hh, int kind, int i, qps_cplx* out, int* rows, int* cols) {
    return guarded(const_cast<qps_ctx*>(hh), [&](Ctx& c) {
        need_device(c);
        const Dims& D = c.dims;
        const int I = D.I, nb = D.nb, P = D.P;
        const size_t nb2 = size_t(nb) * nb;
        auto rng = [&](int lo, int hi) { need(i >= lo && i < hi, "block index out of range"); };
        if (kind < 32) {
            need(c.sys_valid, "assemble_system first (the one-shot path overwrites A with A')");
            switch (kind) {
                case QPS_BLK_A_DIAG: rng(0, I); return get_block(c, c.Adiag.p + i * nb2, nb, 2 * D.N[i], 2 * D.N[i], out, rows, cols);
                case QPS_BLK_A_SUPER: rng(0, I - 1); return get_block(c, c.Asup.p + i * nb2, nb, 2 * D.N[i], 2 * D.N[i + 1], out, rows, cols);
                case QPS_BLK_A_SUB: rng(0, I - 1); return get_block(c, c.Asub.p + i * nb2, nb, 2 * D.N[i + 1], 2 * D.N[i], out, rows, cols);
                case QPS_BLK_B_SELF: rng(0, I); return get_block(c, c.Bself.p + size_t(i) * nb * P, nb, 2 * D.N[i], P, out, rows, cols);
                case QPS_BLK_B_BELOW: rng(0, I); return get_block(c, c.Bbelow.p + size_t(i) * nb * P, nb, 2 * D.N[i], P, out, rows, cols);
                case QPS_BLK_C_SELF:
                    rng(0, I + 1);
                    if (i == I) return zero_block(rows, cols);
                    if (i == 0) return get_block(c, c.Rc.p, D.mC, D.mI, 2 * D.N[0], out, rows, cols);
                    return get_block(c, c.Rint.p + size_t(i - 1) * D.mI * 2 * nb + size_t(nb) * D.mI, D.mI, D.mI, 2 * D.N[i], out, rows, cols);
                case QPS_BLK_C_ABOVE:
                    rng(0, I + 1);
                    if (i == 0) return zero_block(rows, cols);
                    if (i == I) return get_block(c, c.Rc.p + size_t(D.mC) * nb, D.mC, D.mI, 2 * D.N[I - 1], out, rows, cols);
                    return get_block(c, c.Rint.p + size_t(i - 1) * D.mI * 2 * nb, D.mI, D.mI, 2 * D.N[i - 1], out, rows, cols);
                case QPS_BLK_Q:
                    rng(0, I + 1);
                    if (i == 0) return get_block(c, c.Qc.p, D.mC, D.mI, P, out, rows, cols);
                    if (i == I) return get_block(c, c.Qc.p + size_t(D.mC) * D.pC, D.mC, D.mI, P, out, rows, cols);
                    return get_block(c, c.Qint.p + size_t(i - 1) * D.mI * P, D.mI, D.mI, P, out, rows, cols);
                case QPS_BLK_Z_U: return get_block(c, c.Rc.p + D.mI, D.mC, 2 * D.M, 2 * D.N[0], out, rows, cols);
                case QPS_BLK_Z_D: return get_block(c, c.Rc.p + size_t(D.mC) * nb + D.mI, D.mC, 2 * D.M, 2 * D.N[I - 1], out, rows, cols);
                case QPS_BLK_V_U: return get_block(c, c.Qc.p + D.mI, D.mC, 2 * D.M, P, out, rows, cols);
                case QPS_BLK_V_D: return get_block(c, c.Qc.p + size_t(D.mC) * D.pC + D.mI, D.mC, 2 * D.M, P, out, rows, cols);
                case QPS_BLK_W_U: return get_block(c, c.Qc.p + size_t(P) * D.mC + D.mI, D.mC, 2 * D.M, D.nrb, out, rows, cols);
                case QPS_BLK_W_D: return get_block(c, c.Qc.p + size_t(D.mC) * D.pC + size_t(P) * D.mC + D.mI, D.mC, 2 * D.M, D.nrb, out, rows, cols);
                case QPS_BLK_F: return get_block(c, c.f.p, nb, 2 * D.N[0], 1, out, rows, cols);
                case QPS_BLK_CP_FIRST: return get_block(c, c.Rc.p, D.mC, D.mC, 2 * D.N[0], out, rows, cols);
                case QPS_BLK_CP_LAST: return get_block(c, c.Rc.p + size_t(D.mC) * nb, D.mC, D.mC, 2 * D.N[I - 1], out, rows, cols);
                case QPS_BLK_QP_FIRST: return get_block(c, c.Qc.p, D.mC, D.mC, D.pC, out, rows, cols);
                case QPS_BLK_QP_LAST: return get_block(c, c.Qc.p + size_t(D.mC) * D.pC, D.mC, D.mC, D.pC, out, rows, cols);
                case QPS_BLK_BP_FIRST:
                case QPS_BLK_BP_LAST: {
                    const int j = kind == QPS_BLK_BP_FIRST ? 0 : I - 1;
                    const int r = 2 * D.N[j];
                    if (rows) *rows = r;
                    if (cols) *cols = D.pC;
                    if (!out) return;
                    std::memset(out, 0, sizeof(qps_cplx) * size_t(r) * D.pC);
                    const cplx* src = (kind == QPS_BLK_BP_FIRST ? c.Bself.p : c.Bbelow.p) + size_t(j) * nb * P;
                    return get_block(c, src, nb, r, P, out, nullptr, nullptr);
                }
                default: fail(QPS_ERR_USAGE, "unknown block kind");
            }
        }
        need(c.ps_valid, "schur_complement first (block_lu_solve overwrites A')");
        const cplx* Ad = c.ps_separate ? c.Apdiag.p : c.Adiag.p;
        const cplx* Au = c.ps_separate ? c.Apsup.p : c.Asup.p;
        const cplx* Al = c.ps_separate ? c.Apsub.p : c.Asub.p;
        switch (kind) {
            case QPS_BLK_AP_DIAG: rng(0, I); return get_block(c, Ad + i * nb2, nb, 2 * D.N[i], 2 * D.N[i], out, rows, cols);
            case QPS_BLK_AP_SUPER: rng(0, I - 1); return get_block(c, Au + i * nb2, nb, 2 * D.N[i], 2 * D.N[i + 1], out, rows, cols);
            case QPS_BLK_AP_SUB: rng(0, I - 1); return get_block(c, Al + i * nb2, nb, 2 * D.N[i + 1], 2 * D.N[i], out, rows, cols);
            case QPS_BLK_X_FIRST: return get_block(c, c.Xc.p, D.pC, D.pC, 2 * D.N[0], out, rows, cols);
            case QPS_BLK_X_LAST: return get_block(c, c.Xc.p + size_t(D.pC) * nb, D.pC, D.pC, 2 * D.N[I - 1], out, rows, cols);
            case QPS_BLK_X_ABOVE:
                rng(0, I);
                if (i == 0) return zero_block(rows, cols);
                return get_block(c, c.Xint.p + size_t(i - 1) * P * 2 * nb, P, P, 2 * D.N[i - 1], out, rows, cols);
            case QPS_BLK_X_SELF:
                rng(0, I);
                if (i == 0) return zero_block(rows, cols);
                return get_block(c, c.Xint.p + size_t(i - 1) * P * 2 * nb + size_t(nb) * P, P, P, 2 * D.N[i], out, rows, cols);
            default: fail(QPS_ERR_USAGE, "unknown block kind");
        }
    });
}

int qps_fill_evals(const qps_ctx* h, uint64_t* reference, uint64_t* performed) {
    if (!h) return QPS_ERR_USAGE;
    if (reference) *reference = h->c.ref_evals;
    if (performed) *performed = h->c.performed_evals;
    return QPS_OK;
}

int qps_get_phase_times(const qps_ctx* h, qps_phase_times* t) {
    if (!h || !t) return QPS_ERR_USAGE;
    *t = h->c.times;
    return QPS_OK;
}

int qps_solver_diagnostics(const qps_ctx* h, qps_solver_diag* d) {
    if (!h || !d) return QPS_ERR_USAGE;
    d->bcr_path = h->c.bcr_path;
    d->lr_rank_max = h->c.lr_rank_max;
    d->lr_probe_worst = h->c.lr_probe_worst;
    d->refine_steps = h->c.refine_used;
    double nr[3] = {0, 0, 0};  // sqrt of the sums of the per-block squared norms
    const int nbk = h->c.refine_used ? h->c.ref_nrm_n : 0;
    for (int q = 0; q < 3; ++q) {
        for (int b = 0; b < nbk; ++b) nr[q] += h->c.ref_nrm_h[size_t(q) * nbk + b] * h->c.ref_nrm_h[size_t(q) * nbk + b];
        nr[q] = std::sqrt(nr[q]);
    }
    d->refine_res0 = nr[2] > 0 ? nr[0] / nr[2] : 0.0;
    d->refine_res1 = nr[2] > 0 ? nr[1] / nr[2] : 0.0;
    d->lr_width = h->c.bcr_path ? h->c.lr_r : 0;
    d->lr_width_retry = h->c.lr_width_retried ? 1 : 0;
    return QPS_OK;
}

int qps_hankel01(qps_ctx* h, int n, const double* x, qps_cplx* h0, qps_cplx* h1) {
    return guarded(h, [&](Ctx& c) {
        need_device(c);
        for (int i = 0; i < n; ++i)
            if (!(x[i] > 0.0) || !std::isfinite(x[i]))
                fail(QPS_ERR_DOMAIN, "hankel01: argument must be finite and > 0");
        if (n == 0) return;
        DBuf<double> dx;
        DBuf<cplx> d0, d1;
        dx.ensure(n);
        d0.ensure(n);
        d1.ensure(n);
        QPS_CUDA(cudaMemcpyAsync(dx.p, x, sizeof(double) * n, cudaMemcpyHostToDevice, c.stream));
        launch_hankel_batch(n, dx.p, d0.p, d1.p, c.stream);
        QPS_CUDA(cudaMemcpyAsync(h0, d0.p, sizeof(cplx) * n, cudaMemcpyDeviceToHost, c.stream));
        QPS_CUDA(cudaMemcpyAsync(h1, d1.p, sizeof(cplx) * n, cudaMemcpyDeviceToHost, c.stream));
        QPS_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int qps_qsolve(qps_ctx* h, int m, int p, int n, const qps_cplx* Q, const qps_cplx* R, qps_cplx* X, int* rank) {
    return guarded(h, [&](Ctx& c) {
        need_device(c);
        need(m >= p, "qsolve: Q must have at least as many rows as columns");
        need(m > 0 && p > 0 && n > 0, "qsolve: empty operand");
        DBuf<cplx> dQ, dR, dX;
        dQ.ensure(size_t(m) * p);
        dR.ensure(size_t(m) * n);
        dX.ensure(size_t(p) * n);
        QPS_CUDA(cudaMemcpyAsync(dQ.p, Q, sizeof(cplx) * m * p, cudaMemcpyHostToDevice, c.stream));
        QPS_CUDA(cudaMemcpyAsync(dR.p, R, sizeof(cplx) * size_t(m) * n, cudaMemcpyHostToDevice, c.stream));
        CodSet cs;
        cs.ensure(1, m, p, n);
        double lsq = 0;
        qsolve_family_public(c, cs, dQ.p, dR.p, m, size_t(m) * n, dX.p, p, size_t(p) * n, &lsq);
        QPS_CUDA(cudaMemcpyAsync(X, dX.p, sizeof(cplx) * size_t(p) * n, cudaMemcpyDeviceToHost, c.stream));
        if (rank) QPS_CUDA(cudaMemcpyAsync(rank, cs.rank.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
        QPS_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int qps_debug_zgemm(qps_ctx* h, int M, int N, int K, const qps_cplx* A, const qps_cplx* B, qps_cplx* Cm) {
    return guarded(h, [&](Ctx& c) {
        need_device(c);
        DBuf<cplx> dA, dB, dC;
        dA.ensure(size_t(M) * K);
        dB.ensure(size_t(K) * N);
        dC.ensure(size_t(M) * N);
        QPS_CUDA(cudaMemcpyAsync(dA.p, A, sizeof(cplx) * size_t(M) * K, cudaMemcpyHostToDevice, c.stream));
        QPS_CUDA(cudaMemcpyAsync(dB.p, B, sizeof(cplx) * size_t(K) * N, cudaMemcpyHostToDevice, c.stream));
        std::vector<GemmTask> t(1, GemmTask{});
        t[0].nseg = 1;
        t[0].A[0] = dA.p; t[0].lda[0] = M; t[0].B[0] = dB.p; t[0].ldb[0] = K; t[0].K[0] = K;
        t[0].C = dC.p; t[0].ldc = M;
        zgemm_batched(M, N, cplx{1, 0}, cplx{0, 0}, t, c.stream, c.ws.gemm_tasks);
        QPS_CUDA(cudaMemcpyAsync(Cm, dC.p, sizeof(cplx) * size_t(M) * N, cudaMemcpyDeviceToHost, c.stream));
        QPS_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int qps_prof_enable(qps_ctx* h, int on) {
    return guarded(h, [&](Ctx&) { prof_enable(on != 0); });
}

int qps_prof_reset(qps_ctx* h) {
    return guarded(h, [&](Ctx& c) {
        if (!c.host_only) QPS_CUDA(cudaStreamSynchronize(c.stream));
        prof_reset();
        g_h2d_bytes = 0;
        g_d2h_bytes = 0;
    });
}

int qps_prof_stats(qps_ctx* h, int cap, char* names, uint64_t* launches, double* ms, double* flops, double* bytes,
                   double* units) {
    if (!h) return -1;
    if (!h->c.host_only) cudaStreamSynchronize(h->c.stream);
    std::vector<ProfStat> st(cap > 0 ? cap : 0);
    const int n = prof_query(st.data(), cap);
    for (int i = 0; i < std::min(n, cap); ++i) {
        if (names) {
            std::strncpy(names + 64 * i, st[i].name, 63);
            names[64 * i + 63] = 0;
        }
        if (launches) launches[i] = st[i].launches;
        if (ms) ms[i] = st[i].ms;
        if (flops) flops[i] = st[i].flops;
        if (bytes) bytes[i] = st[i].bytes;
        if (units) units[i] = st[i].units;
    }
    return n;
}

uint64_t qps_launch_count(void) { return g_launches.load(); }

int qps_transfer_bytes(const qps_ctx* h, uint64_t* h2d, uint64_t* d2h) {
    if (!h) return QPS_ERR_USAGE;
    if (h2d) *h2d = g_h2d_bytes.load();
    if (d2h) *d2h = g_d2h_bytes.load();
    return QPS_OK;
}

// FP64 peak microbenchmarks for the roofline denominators (north star:
// "FP64 peak measured by a microbenchmark in the same run")
int qps_measure_fp64_peaks(qps_ctx* h, double* dfma_tflops, double* dmma_tflops) {
    return guarded(h, [&](Ctx& c) {
        need_device(c);
        if (dfma_tflops) *dfma_tflops = measure_dfma_tflops(c.stream);
        if (dmma_tflops) *dmma_tflops = measure_dmma_tflops(c.stream);
    });
}

}  // extern "C"
