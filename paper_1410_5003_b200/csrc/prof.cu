#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "prof.h"
#include "qps_internal.h"

namespace qpsb {

std::atomic<uint64_t> g_launches{0};
std::atomic<uint64_t> g_h2d_bytes{0}, g_d2h_bytes{0};

namespace {
struct StagingRing {
    static constexpr size_t kSize = size_t(64) << 20;
    std::mutex mu;
    char* base = nullptr;
    size_t head = 0;
    struct Pending {
        size_t lo, hi;
        cudaEvent_t ev;
    };
    std::deque<Pending> pending;
    std::vector<cudaEvent_t> free_events;
};
StagingRing& ring() {
    static StagingRing* r = new StagingRing();  // never destroyed: outlives every context
    return *r;
}
}  // namespace

void h2d_staged(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return;
    StagingRing& R = ring();
    const size_t need = (bytes + 255) & ~size_t(255);
    if (need > R.kSize / 4) {  // large one-off copies: plain (synchronising) path
        QPS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        return;
    }
    std::lock_guard<std::mutex> lk(R.mu);
    if (!R.base) QPS_CUDA(cudaMallocHost(reinterpret_cast<void**>(&R.base), R.kSize));
    if (R.head + need > R.kSize) R.head = 0;
    const size_t lo = R.head, hi = R.head + need;
    // wait for earlier copies still reading [lo, hi)
    for (auto it = R.pending.begin(); it != R.pending.end();) {
        const bool overlap = it->lo < hi && lo < it->hi;
        if (overlap || cudaEventQuery(it->ev) == cudaSuccess) {
            if (overlap) QPS_CUDA(cudaEventSynchronize(it->ev));
            R.free_events.push_back(it->ev);
            it = R.pending.erase(it);
        } else {
            ++it;
        }
    }
    std::memcpy(R.base + lo, src, bytes);
    QPS_CUDA(cudaMemcpyAsync(dst, R.base + lo, bytes, cudaMemcpyHostToDevice, s));
    cudaEvent_t ev;
    if (R.free_events.empty()) QPS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    else { ev = R.free_events.back(); R.free_events.pop_back(); }
    QPS_CUDA(cudaEventRecord(ev, s));
    R.pending.push_back({lo, hi, ev});
    R.head = hi;
}

namespace {
struct Pending {
    std::string name;
    cudaStream_t s;
    cudaEvent_t e0, e1;
    double flops, bytes, units;
    int nlaunch;
};
struct Agg {
    uint64_t launches = 0;
    double ms = 0, flops = 0, bytes = 0, units = 0;
};
bool g_on = false;
const char* g_phase = nullptr;
std::vector<Pending> g_pending;
std::map<std::string, Agg> g_agg;
std::vector<cudaEvent_t> g_free;
// QPS_PROF_TIMELINE: every scope's [start, end] on its stream, relative to the
// first scope after prof_reset, printed to stderr as the scopes resolve
cudaEvent_t g_ref = nullptr;
bool g_ref_set = false;

cudaEvent_t get_event() {
    if (!g_free.empty()) {
        cudaEvent_t e = g_free.back();
        g_free.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

void resolve() {
    static const bool timeline = getenv("QPS_PROF_TIMELINE") != nullptr;
    for (auto& p : g_pending) {
        cudaEventSynchronize(p.e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, p.e0, p.e1);
        if (timeline && g_ref_set) {
            float t0 = 0;
            cudaEventElapsedTime(&t0, g_ref, p.e0);
            fprintf(stderr, "TL %-28s stream %p start %9.3f end %9.3f ms\n", p.name.c_str(), (void*)p.s, t0, t0 + ms);
        }
        Agg& a = g_agg[p.name];
        a.launches += p.nlaunch;
        a.ms += ms;
        a.flops += p.flops;
        a.bytes += p.bytes;
        a.units += p.units;
        g_free.push_back(p.e0);
        g_free.push_back(p.e1);
    }
    g_pending.clear();
}
}  // namespace

void prof_enable(bool on) { g_on = on; }
bool prof_enabled() { return g_on; }
void prof_reset() {
    resolve();
    g_agg.clear();
    g_ref_set = false;
}

ProfScope::ProfScope(const char* name_, cudaStream_t s_, double flops_, double bytes_, double units_, int nl)
    : name(name_), s(s_), flops(flops_), bytes(bytes_), units(units_), nlaunch(nl) {
    if (!g_on) return;
    e0 = get_event();
    e1 = get_event();
    if (!g_ref_set) {
        if (!g_ref) cudaEventCreate(&g_ref);
        cudaEventRecord(g_ref, s);
        g_ref_set = true;
    }
    cudaEventRecord(e0, s);
}

ProfScope::~ProfScope() {
    if (!e0) return;
    cudaEventRecord(e1, s);
    static const bool phases = getenv("QPS_PROF_PHASES") != nullptr;
    std::string key = (phases && g_phase) ? std::string(g_phase) + ":" + name : std::string(name);
    g_pending.push_back({key, s, e0, e1, flops, bytes, units, nlaunch});
    if (g_pending.size() > 4096) resolve();
}

ProfPhase::ProfPhase(const char* tag) : prev(g_phase) { g_phase = tag; }
ProfPhase::~ProfPhase() { g_phase = prev; }

int prof_query(ProfStat* out, int cap) {
    resolve();
    int i = 0;
    for (auto& kv : g_agg) {
        if (i < cap && out) {
            // names are string literals of the launch sites; keep a stable copy
            static std::map<std::string, std::string> keep;
            keep[kv.first] = kv.first;
            out[i] = ProfStat{keep[kv.first].c_str(), kv.second.launches, kv.second.ms, kv.second.flops,
                              kv.second.bytes, kv.second.units};
        }
        ++i;
    }
    return int(g_agg.size());
}

}  // namespace qpsb
