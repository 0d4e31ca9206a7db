// prof.cu -- launch counting and optional per-launch CUDA-event timing of the
// library's kernels, on the stream each kernel is launched on (bench.py reads it
// to report the dominant kernel's live duration).
#include <vector>

#include "blstm.h"
#include "prof.h"

namespace blstm {

static long g_launches = 0;
static int g_prof_on = 0;  // 0 off, 1 categories 0-2, 2 also helper kernels (timeline)
struct ProfRec {
    int cat;
    cudaEvent_t e0, e1;
    cudaStream_t st;
    int a, b, c;
};
static std::vector<ProfRec> g_recs;   // recorded launches since enable
static std::vector<cudaEvent_t> g_pool;
static size_t g_pool_used = 0;
static int g_suspend = 0;
static int g_cat_mask = -1;  // blstm_profile_select

void prof_suspend(int on) { g_suspend += on ? 1 : -1; }

void note_launch(int n) { g_launches += n; }
long launch_count() { return g_launches; }

static cudaEvent_t pool_event() {
    if (g_pool_used == g_pool.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        g_pool.push_back(e);
    }
    return g_pool[g_pool_used++];
}

int prof_begin(int cat, cudaStream_t st, int a, int b, int c) {
    if (!g_prof_on || g_suspend > 0 || (cat == PROF_OTHER && g_prof_on < 2) || !((g_cat_mask >> cat) & 1)) return -1;
    ProfRec r{cat, pool_event(), pool_event(), st, a, b, c};
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
    g_prof_on = on < 0 ? 0 : on;
    g_recs.clear();
    g_pool_used = 0;
    return 0;
}

extern "C" int blstm_profile_select(int cat_mask) {
    g_cat_mask = cat_mask;
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

extern "C" int blstm_profile_timeline(double *rec, int max_recs) {
    if (g_recs.empty()) return 0;
    std::vector<cudaStream_t> streams;
    int n = 0;
    for (const ProfRec &r : g_recs) {
        if (n >= max_recs) break;
        if (cudaEventSynchronize(r.e1) != cudaSuccess) return BLSTM_ERR_CUDA;
        float t0 = 0.f, t1 = 0.f;
        if (cudaEventElapsedTime(&t0, g_recs[0].e0, r.e0) != cudaSuccess) return BLSTM_ERR_CUDA;
        if (cudaEventElapsedTime(&t1, g_recs[0].e0, r.e1) != cudaSuccess) return BLSTM_ERR_CUDA;
        int si = 0;
        while (si < (int)streams.size() && streams[si] != r.st) ++si;
        if (si == (int)streams.size()) streams.push_back(r.st);
        double *o = rec + 7L * n;
        o[0] = r.cat; o[1] = si; o[2] = t0; o[3] = t1; o[4] = r.a; o[5] = r.b; o[6] = r.c;
        ++n;
    }
    return n;
}
