// graph.cu -- capture-once / replay CUDA graphs (graph.h).
#include <map>

#include "gemm.h"
#include "graph.h"
#include "prof.h"

namespace blstm {

namespace {

struct GraphEntry {
    cudaGraphExec_t exec;
    long launches;
};
std::map<std::vector<uint64_t>, GraphEntry> g_graphs;
cudaStream_t g_cap = nullptr;  // the capture stream

int cap_init() {
    if (g_cap) return 0;
    return cudaStreamCreateWithFlags(&g_cap, cudaStreamNonBlocking) == cudaSuccess ? 0 : -5;
}

}  // namespace

int graph_run(const std::vector<uint64_t> &key, int cat, cudaStream_t st, std::initializer_list<const void *> kernels,
              const std::function<int(cudaStream_t)> &body) {
    auto it = g_graphs.find(key);
    if (it == g_graphs.end()) {
        if (gemm_prepare() || cap_init()) return -5;
        cudaFuncAttributes fa;
        for (const void *k : kernels)
            if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) return -5;
        const long n0 = launch_count();
        if (cudaStreamBeginCapture(g_cap, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return -5;
        prof_suspend(1);
        const int rc = body(g_cap);
        prof_suspend(0);
        cudaGraph_t graph = nullptr;
        const cudaError_t e = cudaStreamEndCapture(g_cap, &graph);
        const long nl = launch_count() - n0;
        note_launch((int)-nl);  // counted when the graph runs, not when it is recorded
        if (rc || e != cudaSuccess || !graph) {
            if (graph) cudaGraphDestroy(graph);
            return -5;
        }
        GraphEntry en{nullptr, nl};
        const cudaError_t ei = cudaGraphInstantiate(&en.exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ei != cudaSuccess) return -5;
        it = g_graphs.emplace(key, en).first;
    }
    ProfScope ps(cat, st);
    if (cudaGraphLaunch(it->second.exec, st) != cudaSuccess) return -5;
    note_launch((int)it->second.launches);
    return 0;
}

}  // namespace blstm
