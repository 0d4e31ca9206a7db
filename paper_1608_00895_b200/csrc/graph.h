// graph.h -- capture-once / replay CUDA graphs of launch-bound loops (the step-launched
// recurrence, the MDLSTM wavefront).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <initializer_list>
#include <vector>

namespace blstm {

// Runs body's launches as one CUDA graph on st.  The first call with a given key records body on
// a capture stream of the library's own (capture is not allowed on the legacy default stream) and
// instantiates the graph; later calls with the same key replay it.  key must name every pointer
// and size body bakes into its launches.  kernels: every non-GEMM kernel body launches (loaded
// before capture: a lazy module load synchronizes the context, which capture forbids).  The
// replay is one launch scope of category cat (prof.h).
int graph_run(const std::vector<uint64_t> &key, int cat, cudaStream_t st, std::initializer_list<const void *> kernels,
              const std::function<int(cudaStream_t)> &body);
inline uint64_t u64(const void *p) { return (uint64_t)(uintptr_t)p; }

}  // namespace blstm
