// Launch-to-launch time of a tiny kernel vs the size of its __grid_constant__
// parameter block (the decode kernels pass a 5.8 KB KParams): back-to-back
// launches on one stream, CUDA events around each, median.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o param_launch param_launch.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

template <int N>
struct Blob { unsigned v[N / 4]; };

template <int N>
__global__ void k(const __grid_constant__ Blob<N> b, unsigned* out) {
  if (threadIdx.x == 0) out[blockIdx.x] = b.v[N / 4 - 1] + b.v[0];
}

template <int N>
float run(unsigned* out, int reps) {
  Blob<N> b{};
  b.v[0] = 1;
  cudaStream_t s;
  cudaStreamCreate(&s);
  std::vector<cudaEvent_t> ev(2 * reps);
  for (auto& e : ev) cudaEventCreate(&e);
  for (int i = 0; i < 20; ++i) k<N><<<1, 64, 0, s>>>(b, out);
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(ev[2 * i], s);
    k<N><<<1, 64, 0, s>>>(b, out);
    cudaEventRecord(ev[2 * i + 1], s);
  }
  cudaStreamSynchronize(s);
  std::vector<float> t(reps);
  for (int i = 0; i < reps; ++i) cudaEventElapsedTime(&t[i], ev[2 * i], ev[2 * i + 1]);
  std::sort(t.begin(), t.end());
  return t[reps / 2] * 1e3f;
}

// The same launch captured once into a CUDA graph and replayed.
template <int N>
float run_graph(unsigned* out, int reps) {
  Blob<N> b{};
  b.v[0] = 1;
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  k<N><<<1, 64, 0, s>>>(b, out);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  std::vector<cudaEvent_t> ev(2 * reps);
  for (auto& e : ev) cudaEventCreate(&e);
  for (int i = 0; i < 20; ++i) cudaGraphLaunch(ge, s);
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(ev[2 * i], s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(ev[2 * i + 1], s);
  }
  cudaStreamSynchronize(s);
  std::vector<float> t(reps);
  for (int i = 0; i < reps; ++i) cudaEventElapsedTime(&t[i], ev[2 * i], ev[2 * i + 1]);
  std::sort(t.begin(), t.end());
  return t[reps / 2] * 1e3f;
}

int main() {
  unsigned* out;
  cudaMalloc(&out, 4096);
  printf("param 64 B:   %.2f us\n", run<64>(out, 200));
  printf("param 1 KB:   %.2f us\n", run<1024>(out, 200));
  printf("param 4 KB:   %.2f us\n", run<4096>(out, 200));
  printf("param 5.8 KB: %.2f us\n", run<5808>(out, 200));
  printf("param 16 KB:  %.2f us\n", run<16384>(out, 200));
  printf("param 29 KB:  %.2f us\n", run<29696>(out, 200));
  printf("graph replay, param 64 B:   %.2f us\n", run_graph<64>(out, 200));
  printf("graph replay, param 5.8 KB: %.2f us\n", run_graph<5808>(out, 200));
  return 0;
}
