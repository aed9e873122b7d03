// Microbenchmark: cost of a cooperative-groups grid barrier on one B200 (148 CTAs x T threads),
// and of an empty kernel boundary inside a CUDA graph, for the persistent explicit-iteration design.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ubench_gsync.cu -o tools/ubench_gsync
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_sync(int n, double* sink) {
  cg::grid_group g = cg::this_grid();
  double acc = 0;
  for (int i = 0; i < n; ++i) {
    acc += __ldcg(sink + (blockIdx.x + i) % gridDim.x);
    g.sync();
  }
  if (acc == 12345.0) sink[0] = acc;
}
__global__ void k_empty(double* sink) {
  if (sink[0] == 12345.0) sink[1] = 1;
}
int main() {
  double* sink;
  cudaMalloc(&sink, 4096 * 8);
  cudaMemset(sink, 0, 4096 * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int T : {256, 512, 1024}) {
    const int n = 2000;
    void* args[] = {(void*)&n, (void*)&sink};
    cudaLaunchCooperativeKernel((void*)k_sync, 148, T, args, 0, 0);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_sync, 148, T, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("grid.sync 148 x %4d: %.3f us per barrier (%s)\n", T, ms * 1e3 / n,
           cudaGetErrorString(cudaGetLastError()));
  }
  // graph of 2000 dependent tiny kernels (148 x 256)
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaGraph_t gr;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 2000; ++i) k_empty<<<148, 256, 0, s>>>(sink);
  cudaStreamEndCapture(s, &gr);
  cudaGraphInstantiate(&ge, gr, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEventRecord(a, s);
  cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("graph kernel boundary (148 x 256 empty): %.3f us per kernel\n", ms * 1e3 / 2000);
  return 0;
}
