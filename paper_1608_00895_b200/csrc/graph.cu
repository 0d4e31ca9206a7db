// graph.cu -- capture-once / replay CUDA graphs (graph.h).
//
// The cache is process-global, keyed by (device, caller's key), guarded by a mutex and bounded
// (kMaxGraphs, least recently used evicted).  Each entry remembers an event recorded after its last
// replay; eviction waits for that event before destroying the executable graph, so a graph still
// in flight on some stream is never freed under it.  The capture stream is per device.
#include <list>
#include <map>
#include <mutex>

#include "gemm.h"
#include "graph.h"
#include "prof.h"

namespace blstm {

namespace {

constexpr size_t kMaxGraphs = 48;  // C5: 4 layers x 2 (fwd chain, bwd chain) per workspace, several workspaces

struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    cudaEvent_t done = nullptr;  // recorded after the latest replay
    long launches = 0;
    std::list<std::vector<uint64_t>>::iterator lru;
};
std::mutex g_mu;
std::map<std::vector<uint64_t>, GraphEntry> g_graphs;
std::list<std::vector<uint64_t>> g_lru;  // front = most recently used
std::map<int, cudaStream_t> g_cap;       // per-device capture stream

int cap_stream(int dev, cudaStream_t *out) {
    auto it = g_cap.find(dev);
    if (it != g_cap.end()) {
        *out = it->second;
        return 0;
    }
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return -5;
    g_cap[dev] = s;
    *out = s;
    return 0;
}

void evict_one() {
    const std::vector<uint64_t> &victim = g_lru.back();
    auto it = g_graphs.find(victim);
    if (it != g_graphs.end()) {
        if (it->second.done) {
            cudaEventSynchronize(it->second.done);  // the last replay has finished
            cudaEventDestroy(it->second.done);
        }
        cudaGraphExecDestroy(it->second.exec);
        g_graphs.erase(it);
    }
    g_lru.pop_back();
}

}  // namespace

int graph_run(const std::vector<uint64_t> &key_in, int cat, cudaStream_t st, std::initializer_list<const void *> kernels,
              const std::function<int(cudaStream_t)> &body) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -5;
    std::vector<uint64_t> key;
    key.reserve(key_in.size() + 1);
    key.push_back((uint64_t)dev);
    key.insert(key.end(), key_in.begin(), key_in.end());

    std::lock_guard<std::mutex> lock(g_mu);
    auto it = g_graphs.find(key);
    if (it == g_graphs.end()) {
        cudaStream_t cap = nullptr;
        if (gemm_prepare() || cap_stream(dev, &cap)) return -5;
        cudaFuncAttributes fa;
        for (const void *k : kernels)
            if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) return -5;
        const long n0 = launch_count();
        if (cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return -5;
        prof_suspend(1);
        const int rc = body(cap);
        prof_suspend(0);
        cudaGraph_t graph = nullptr;
        const cudaError_t e = cudaStreamEndCapture(cap, &graph);
        const long nl = launch_count() - n0;
        note_launch((int)-nl);  // counted when the graph runs, not when it is recorded
        if (rc || e != cudaSuccess || !graph) {
            if (graph) cudaGraphDestroy(graph);
            return -5;
        }
        GraphEntry en;
        en.launches = nl;
        const cudaError_t ei = cudaGraphInstantiate(&en.exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ei != cudaSuccess) return -5;
        if (cudaEventCreateWithFlags(&en.done, cudaEventDisableTiming) != cudaSuccess) {
            cudaGraphExecDestroy(en.exec);
            return -5;
        }
        while (g_graphs.size() >= kMaxGraphs && !g_lru.empty()) evict_one();
        g_lru.push_front(key);
        en.lru = g_lru.begin();
        it = g_graphs.emplace(key, en).first;
    } else if (it->second.lru != g_lru.begin()) {
        g_lru.splice(g_lru.begin(), g_lru, it->second.lru);  // most recently used
    }
    ProfScope ps(cat, st);
    if (cudaGraphLaunch(it->second.exec, st) != cudaSuccess) return -5;
    if (cudaEventRecord(it->second.done, st) != cudaSuccess) return -5;
    note_launch((int)it->second.launches);
    return 0;
}

}  // namespace blstm
