// dp.cu -- data parallelism over NCCL (§4.1).
//
// The paper runs one process per GPU; a CPU master holds the parameters, sends an
// "image" to each worker, and after "a specific amount of batches" averages the
// workers' parameters, over sockets with serialized arrays.
// Here the image lives on every GPU and the exchange is an in-place NCCL allreduce
// over NVLink/NVSwitch: SUM of gradients each step (sync mode, one big batch, the
// unscaled-gradient convention of P:253-254) or MEAN of parameters every K steps
// (the paper's averaging).  DESIGN.md R8 / §6.
#include <cstdio>
#include <nccl.h>

#include "blstm.h"

// A 1-rank communicator runs the same NCCL calls (an in-place copy; the average divides by 1):
// the path is exercised by a one-GPU test bit for bit against comm = NULL.
struct dp_comm {
    ncclComm_t comm;
    int nranks, rank;
};

int blstm_set_error(int code, const char *msg);

static int nccl_fail(ncclResult_t r, const char *what) {
    char buf[256];
    snprintf(buf, sizeof(buf), "%s: %s", what, ncclGetErrorString(r));
    return blstm_set_error(BLSTM_ERR_NCCL, buf);
}

extern "C" int dp_get_unique_id(unsigned char id[128]) {
    if (!id) return BLSTM_ERR_ARG;
    ncclUniqueId u;
    ncclResult_t r = ncclGetUniqueId(&u);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    static_assert(sizeof(u.internal) == 128, "ncclUniqueId size");
    for (int i = 0; i < 128; ++i) id[i] = (unsigned char)u.internal[i];
    return 0;
}

extern "C" int dp_comm_init(int nranks, int rank, const unsigned char id[128], dp_comm **out) {
    if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return BLSTM_ERR_ARG;
    ncclUniqueId u;
    for (int i = 0; i < 128; ++i) u.internal[i] = (char)id[i];
    dp_comm *c = new dp_comm;
    c->nranks = nranks;
    c->rank = rank;
    ncclResult_t r = ncclCommInitRank(&c->comm, nranks, u, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_fail(r, "ncclCommInitRank");
    }
    *out = c;
    return 0;
}

int dp_allreduce_grads_impl(dp_comm *c, float *grad, size_t n, cudaStream_t st) {
    if (!c || !grad) return BLSTM_ERR_ARG;
    ncclResult_t r = ncclAllReduce(grad, grad, n, ncclFloat32, ncclSum, c->comm, st);
    return r == ncclSuccess ? 0 : nccl_fail(r, "ncclAllReduce(sum)");
}

extern "C" int dp_allreduce_grads(dp_comm *c, float *grad, size_t n, void *stream) {
    return dp_allreduce_grads_impl(c, grad, n, (cudaStream_t)stream);
}

extern "C" int dp_average_params(dp_comm *c, float *theta, size_t n, void *stream) {
    if (!c || !theta) return BLSTM_ERR_ARG;
    ncclResult_t r = ncclAllReduce(theta, theta, n, ncclFloat32, ncclAvg, c->comm, (cudaStream_t)stream);
    return r == ncclSuccess ? 0 : nccl_fail(r, "ncclAllReduce(avg)");
}

extern "C" int dp_comm_destroy(dp_comm *c) {
    if (!c) return 0;
    ncclResult_t r = ncclCommDestroy(c->comm);
    delete c;
    return r == ncclSuccess ? 0 : nccl_fail(r, "ncclCommDestroy");
}
