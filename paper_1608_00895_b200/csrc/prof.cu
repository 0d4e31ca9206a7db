// prof.cu -- launch counting and optional per-launch CUDA-event timing of the
// library's kernels, on the stream each kernel is launched on (bench.py reads it
// to report the dominant kernel's live duration).
#include <vector>

#include "blstm.h"
#include "prof.h"

namespace blstm {

static long g_launches = 0;
static bool g_prof_on = false;
struct ProfRec {
    int cat;
    cudaEvent_t e0, e1;
};
static std::vector<ProfRec> g_recs;   // recorded launches since enable
static std::vector<cudaEvent_t> g_pool;
static size_t g_pool_used = 0;
static int g_suspend = 0;

void prof_suspend(int on) { g_suspend += on ? 1 : -1; }

void note_launch(int n) { g_launches += n; }

static cudaEvent_t pool_event() {
    if (g_pool_used == g_pool.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        g_pool.push_back(e);
    }
    return g_pool[g_pool_used++];
}

int prof_begin(int cat, cudaStream_t st) {
    if (!g_prof_on || g_suspend > 0) return -1;
    ProfRec r{cat, pool_event(), pool_event()};
    if (!r.e0 || !r.e1) return -1;
    cudaEventRecord(r.e0, st);
    g_recs.push_back(r);
    return (int)g_recs.size() - 1;
}
void prof_end(int idx, cudaStream_t st) {
    if (idx < 0 || !g_prof_on) return;
    cudaEventRecord(g_recs[idx].e1, st);
}

}  // namespace blstm

using namespace blstm;

extern "C" long blstm_launch_count(void) { return g_launches; }

extern "C" int blstm_profile_enable(int on) {
    g_prof_on = on != 0;
    g_recs.clear();
    g_pool_used = 0;
    return 0;
}

extern "C" int blstm_profile_read(int cat, double *total_ms, long *launches) {
    double tot = 0.0;
    long n = 0;
    for (const ProfRec &r : g_recs) {
        if (r.cat != cat) continue;
        if (cudaEventSynchronize(r.e1) != cudaSuccess) return BLSTM_ERR_CUDA;
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, r.e0, r.e1) != cudaSuccess) return BLSTM_ERR_CUDA;
        tot += ms;
        ++n;
    }
    if (total_ms) *total_ms = tot;
    if (launches) *launches = n;
    return 0;
}
