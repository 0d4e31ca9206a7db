// optim.h -- internal interface of the update-rule kernels (optim.cu).
#pragma once
#include <cuda_runtime.h>

namespace blstm {

enum { OPT_SGD = 0, OPT_MOMENTUM = 1, OPT_NESTEROV = 2, OPT_ADAGRAD = 3, OPT_ADADELTA = 4, OPT_ADAM = 5 };

struct OptArgs {
    float lr, mu, rho, b1, b2, eps, l2, max_norm;
    float rho1, b1c, b2c;  // 1-rho, 1-b1, 1-b2 (host-computed in fp64, then rounded once)
    float c1, c2;          // Adam bias corrections 1/(1 - b1^t), 1/(1 - b2^t) (host fp64)
};

// Sorted element boundaries of the bias ranges [bnd[2k], bnd[2k+1]); unused slots hold LONG_MAX.
// An index is a bias entry iff an odd number of boundaries is <= it.  nb == 0: no bias entries.
constexpr int OPT_MAX_BOUNDS = 128;
struct OptBiasTable {
    int nb;
    long bnd[OPT_MAX_BOUNDS];
};

// fp64 partials the norm pass writes (workspace of opt_norm_partials() doubles)
int opt_norm_partials();
// s0 / s1: the rule's state (NULL where unused); all pointers 16-byte aligned.
int opt_update(int rule, float *theta, float *grad, float *s0, float *s1, long n, const OptArgs &a,
               double max_norm, const OptBiasTable &tab, double *partial, int zero, cudaStream_t st);

constexpr int MAX_REPLICAS = 16;
struct ReplicaPtrs {
    float *p[MAX_REPLICAS];
};
// x_r <- scale * sum_{q<n} x_q for r < n (fixed order; every replica gets identical bits);
// pointers 16-byte aligned
int reduce_replicas(const ReplicaPtrs &rp, int n, long len, float scale, cudaStream_t st);

}  // namespace blstm
