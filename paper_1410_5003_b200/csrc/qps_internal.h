// Internal declarations of the B200 implementation of the qpscat hot path.
// Host code is C++17; device code targets sm_100a only.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "qpscat_b200.h"

namespace qpsb {

// host<->device traffic counters (bench.py's e2e bytes per step)
extern std::atomic<uint64_t> g_h2d_bytes, g_d2h_bytes;

// Stream-ordered host->device copy through a pinned staging ring: the source
// is copied into page-locked memory and the DMA is queued without waiting for
// the stream (a pageable cudaMemcpyAsync would synchronise it, serialising the
// host with every small task-table upload of a launch chain).
void h2d_staged(void* dst, const void* src, size_t bytes, cudaStream_t s);

// ---------------------------------------------------------------------------
// Error taxonomy (mirrors /root/reference/proj/include/qpscat/errors.hpp:9-40)
// ---------------------------------------------------------------------------
struct Error : std::runtime_error {
    int status;
    int layer;
    uint64_t bytes;
    Error(int st, const std::string& msg, int layer_ = 0, uint64_t bytes_ = 0)
        : std::runtime_error(msg), status(st), layer(layer_), bytes(bytes_) {}
};
[[noreturn]] inline void fail(int st, const std::string& msg) { throw Error(st, msg); }
// internal: the block solve must be re-run with the dense reduction (bcr_solve)
constexpr const char* kRetryDense = "qpsb: retry with the dense cyclic reduction";
// the adaptive (truncated) coupling bases failed the a-posteriori probe after the
// early level-0 factorization: once more with the full basis width
constexpr const char* kRetryWidth = "qpsb: retry with the full low-rank basis width";

// counted device->host copy
#define QPS_D2H(dst, src, bytes, stream)                                                   \
    do {                                                                                   \
        QPS_CUDA(cudaMemcpyAsync((dst), (src), (bytes), cudaMemcpyDeviceToHost, (stream)));  \
        ::qpsb::g_d2h_bytes += (bytes);                                                    \
    } while (0)

#define QPS_CUDA(call)                                                                          \
    do {                                                                                        \
        cudaError_t qps_e_ = (call);                                                            \
        if (qps_e_ != cudaSuccess)                                                              \
            throw ::qpsb::Error(QPS_ERR_CUDA, std::string(#call " failed: ") +                  \
                                                  cudaGetErrorString(qps_e_) + " at " __FILE__); \
    } while (0)

constexpr double kPi = 3.14159265358979323846;  // types.hpp:14

// ---------------------------------------------------------------------------
// Device memory
// ---------------------------------------------------------------------------
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void ensure(size_t count) {
        if (count <= n && p) return;
        release();
        if (count == 0) return;
        QPS_CUDA(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    void upload(const std::vector<T>& h, cudaStream_t s) {
        ensure(h.size());
        if (!h.empty()) {
            h2d_staged(p, h.data(), h.size() * sizeof(T), s);
            g_h2d_bytes += h.size() * sizeof(T);
        }
    }
    void zero(cudaStream_t s) {
        if (p && n) QPS_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
    }
};

// Pinned host buffer: small device->host reads that must not block the host
// (a D2H copy into pageable memory returns only once the stream reaches it).
template <class T>
struct HBuf {
    T* p = nullptr;
    size_t n = 0;
    HBuf() = default;
    HBuf(const HBuf&) = delete;
    HBuf& operator=(const HBuf&) = delete;
    ~HBuf() {
        if (p) cudaFreeHost(p);
    }
    void ensure(size_t count) {
        if (count <= n && p) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = 0;
        if (count == 0) return;
        QPS_CUDA(cudaMallocHost(reinterpret_cast<void**>(&p), count * sizeof(T)));
        n = count;
    }
    T& operator[](size_t i) { return p[i]; }
    const T& operator[](size_t i) const { return p[i]; }
};

// ---------------------------------------------------------------------------
// Host geometry (reference-equivalent arithmetic; geometry.hpp)
// ---------------------------------------------------------------------------
enum SegKind : int { SEG_SINE = 0, SEG_FOURIER = 1, SEG_LINE = 2 };

// Device-evaluable description of one quadrature segment (QuadSegment,
// geometry.hpp:73-78): the std::function closures of the reference become data.
struct SegDesc {
    int kind;        // SegKind
    int n;           // node count
    int offset;      // first node in the interface
    int periodic;    // 1 for a periodic-smooth interface
    int q;           // Kress grading exponent (lines)
    int ncos, nsin;  // Fourier coefficient counts
    int coef_off;    // offset into the Fourier coefficient pool
    double d, y0, amp, phase;  // period, offset height, sine parameters
    double Ax, Ay, Bx, By;     // line end points
};

struct HostInterface {
    std::vector<double> x, y, nx, ny, w, speed;
    std::vector<SegDesc> segs;
    // open-arc (graded-corner) interfaces: the Alpert auxiliary nodes of every
    // row, computed on the host with the reference's arithmetic (the device's
    // pow/sincos would move nodes that sit 8e-4 h from a target near a corner
    // by a few ulps, ~1e-9 of the self-block entries): per row 2 x 15 entries
    // of (x, y, n_x, n_y, quadrature weight h w_k |Z'|), side -1 then +1
    std::vector<double> aux;
    double y_min = 0, y_max = 0, wall_y = 0;
    bool smooth = false;
    int N() const { return int(x.size()); }
};

struct StackDesc {
    double d = 1.0;
    std::vector<double> eps, mu;
    std::vector<qps_interface_spec> ifaces;  // pointers into the arrays below
    std::vector<std::vector<double>> cosc, sinc, verts;
    std::vector<std::vector<int>> nodes;
};

struct HostGeometry {
    double d = 1.0;
    int I = 0;
    std::vector<HostInterface> ifaces;
    double y_U = 0, y_D = 0;
    std::vector<double> wall_lo, wall_hi;
    std::vector<std::vector<double>> wall_ys;  // I+1 x Mw
    std::vector<double> ud_x;                  // M
    std::vector<double> pc_x, pc_y;            // proxy centres, I+1
    std::vector<std::vector<double>> px, py, pnx, pny;  // I+1 x P
    std::vector<double> fourier_pool;
    int P = 0, Mw = 0, M = 0;
    double R = 0;
};

struct Numerics {
    int P = 60, Mw = 120, M = 60, K = 0;
    double R = 2.0;
    int grading_q = 6;
    double clearance = 0.05;
    uint64_t memory_budget = uint64_t(4) << 30;
};

HostGeometry build_geometry(const StackDesc& st, const Numerics& num);
// build_interface_geometry (geometry.hpp:423-447): one interface's quadrature
HostInterface build_interface_geometry(const qps_interface_spec& sp, double d);

struct Problem {
    double omega = 0, theta = 0;
    std::vector<double> k;
    double ar = 1, ai = 0;  // alpha
    int K = 0;
    double kappa(int n, double d) const;
};
Problem make_problem(const StackDesc& st, const HostGeometry& g, double omega, double theta, int K);
int choose_rb_order(const StackDesc& st, const HostGeometry& g, double omega, double theta);

// classify_point (postprocess.hpp:27-39): region 0 above y_U, 1 layer, 2 below y_D
int classify_point(const StackDesc& st, const HostGeometry& g, double x, double y, int* layer);

// reference fill count, ShiftBlockCache::fill_evals (assembly.hpp:285)
uint64_t reference_fill_evals(const HostGeometry& g);

}  // namespace qpsb
