// prof.h -- internal launch counting / event timing (prof.cu).
#pragma once
#include <cuda_runtime.h>

namespace blstm {

enum { PROF_REC_FWD = 0, PROF_REC_BWD = 1, PROF_GEMM = 2, PROF_OTHER = 3 };

void note_launch(int n = 1);
long launch_count();
// a, b, c: launch shape recorded for the timeline (GEMM: M, N, K)
int prof_begin(int cat, cudaStream_t st, int a = 0, int b = 0, int c = 0);
void prof_end(int idx, cudaStream_t st);

// while > 0, prof_begin records nothing (a launch pair timed as one scope: an event between a
// primary kernel and its programmatic dependent would serialize them)
void prof_suspend(int on);

// RAII bracket of one launch
struct ProfScope {
    int idx;
    cudaStream_t st;
    ProfScope(int cat, cudaStream_t s, int a = 0, int b = 0, int c = 0) : idx(prof_begin(cat, s, a, b, c)), st(s) {}
    ~ProfScope() { prof_end(idx, st); }
};

}  // namespace blstm
