// Probe: CUDA graph with a conditional WHILE node whose body holds two
// cooperative kernels (grid.sync inside), the loop condition set from device
// code.  Build: nvcc -gencode arch=compute_100a,code=sm_100a cond_graph.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cont(int* ctr, int* log, int limit, cudaGraphConditionalHandle h) {
  cg::grid_group g = cg::this_grid();
  g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int c = ++ctr[0];
    log[c] = 1000 + ctr[1];
    cudaGraphSetConditional(h, c < limit ? 1u : 0u);
  }
}
__global__ void k_sweep(int* ctr) {
  cg::grid_group g = cg::this_grid();
  if (threadIdx.x == 0) atomicAdd(ctr + 1, 1);
  g.sync();
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int *ctr, *log; CK(cudaMalloc(&ctr, 64)); CK(cudaMalloc(&log, 4096));
  cudaStream_t s; CK(cudaStreamCreate(&s));
  cudaGraph_t g; CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault));
  int limit = 5;
  dim3 grid(2 * nsm), blk(256);
  void* a0[] = {&ctr, &log, &limit, &h};
  void* a1[] = {&ctr};
  CK(cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  CK(cudaLaunchCooperativeKernel((void*)k_cont, grid, blk, a0, 0, s));
  CK(cudaStreamEndCapture(s, &g));
  size_t nn = 0; CK(cudaGraphGetNodes(g, nullptr, &nn));
  cudaGraphNode_t first; nn = 1; CK(cudaGraphGetNodes(g, &first, &nn));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cn;
  CK(cudaGraphAddNode(&cn, g, &first, 1, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  CK(cudaLaunchCooperativeKernel((void*)k_sweep, grid, blk, a1, 0, s));
  CK(cudaLaunchCooperativeKernel((void*)k_cont, grid, blk, a0, 0, s));
  CK(cudaStreamEndCapture(s, &body));
  cudaGraphExec_t ex; CK(cudaGraphInstantiate(&ex, g, 0));
  for (int rep = 0; rep < 3; ++rep) {
    CK(cudaMemsetAsync(ctr, 0, 64, s));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    CK(cudaGraphLaunch(ex, s));
    cudaEventRecord(e1, s);
    CK(cudaStreamSynchronize(s));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int hc[2]; CK(cudaMemcpy(hc, ctr, 8, cudaMemcpyDeviceToHost));
    printf("rep %d: conts %d sweeps-atomics %d (expect %d conts, %d x %d), %.1f us\n", rep, hc[0], hc[1],
           limit, limit - 1, 2 * nsm, ms * 1e3);
  }
  printf("OK\n");
  return 0;
}
