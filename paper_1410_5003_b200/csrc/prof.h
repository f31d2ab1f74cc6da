// Kernel-family instrumentation: launch counting (always on) and, when
// enabled, CUDA-event timing of every launch on the stream it runs on,
// together with the algorithmic FLOPs / bytes / kernel evaluations of that
// launch.  bench.py reads these to report achieved rates of the dominant
// kernel over the timed region.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

namespace qpsb {

extern std::atomic<uint64_t> g_launches;
// every kernel launch site of the library counts itself (qps_launch_count)
#define QPS_NOTE_LAUNCH() (::qpsb::g_launches.fetch_add(1, std::memory_order_relaxed))

void prof_enable(bool on);
bool prof_enabled();
void prof_reset();
// name must be a string literal (stored by pointer)
struct ProfScope {
    const char* name;
    cudaStream_t s;
    double flops, bytes, units;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    int nlaunch;
    ProfScope(const char* name_, cudaStream_t s_, double flops_, double bytes_ = 0.0, double units_ = 0.0,
              int nlaunch_ = 1);
    ~ProfScope();
};
// aggregate stats; returns number of families, fills at most cap entries
struct ProfStat {
    const char* name;
    uint64_t launches;
    double ms, flops, bytes, units;
};
int prof_query(ProfStat* out, int cap);
// with QPS_PROF_PHASES set, families are keyed "phase:name" inside a ProfPhase
struct ProfPhase {
    const char* prev;
    explicit ProfPhase(const char* tag);
    ~ProfPhase();
};

}  // namespace qpsb
