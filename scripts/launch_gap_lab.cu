// Launch-gap micro-lab (standalone): back-to-back kernels of a fixed spin
// length, with and without programmatic dependent launch, in a stream and in
// a CUDA graph.  Shows how kernel boundaries round kernel durations.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/launch_gap_lab.cu -o build/launch_gap_lab
#include <cuda_runtime.h>
#include <stdio.h>

__global__ void spin(long long cycles, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
}

static void launch(cudaStream_t s, long long cyc, int blocks, int pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(128);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, spin, cyc, pdl);
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 200;
  for (int blocks : {1, 148, 592}) {
    for (long long cyc : {0LL, 1000LL, 2000LL, 3000LL, 4000LL, 6000LL, 8000LL, 12000LL}) {
      float res[4];
      for (int mode = 0; mode < 4; ++mode) {  // 0 stream, 1 stream+PDL, 2 graph, 3 graph+PDL
        const int pdl = mode & 1;
        cudaGraphExec_t ge = nullptr;
        if (mode >= 2) {
          cudaGraph_t g;
          cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
          for (int i = 0; i < reps; ++i) launch(s, cyc, blocks, pdl);
          cudaStreamEndCapture(s, &g);
          cudaGraphInstantiate(&ge, g, 0);
          cudaGraphLaunch(ge, s);
        } else {
          for (int i = 0; i < 10; ++i) launch(s, cyc, blocks, pdl);
        }
        cudaStreamSynchronize(s);
        spin<<<1, 1, 0, s>>>(20000000LL, 0);
        cudaEventRecord(a, s);
        if (mode >= 2) cudaGraphLaunch(ge, s);
        else
          for (int i = 0; i < reps; ++i) launch(s, cyc, blocks, pdl);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        res[mode] = ms * 1e3f / reps;
      }
      printf("blocks %4d spin %6lld cyc (%.2f us): stream %.2f  stream+pdl %.2f  graph %.2f  graph+pdl %.2f us/kernel\n",
             blocks, cyc, cyc / 1965.0, res[0], res[1], res[2], res[3]);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
