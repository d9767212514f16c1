// nccl_ce_test.cu — probe: NCCL all-gather of one 1B-fragment payload per GPU,
// default vs symmetric window + NCCL_CTA_POLICY_ZERO (copy engines), while a
// bandwidth-heavy kernel runs on another stream (the contention question).
// Single process, all visible GPUs.  Not part of the product.
#include <cuda_runtime.h>
#include <nccl.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
#define NK(x) do { ncclResult_t r = (x); if (r != ncclSuccess) { printf("NCCL %s @%d\n", ncclGetErrorString(r), __LINE__); exit(1);} } while (0)

__global__ void stream_kernel(const float4* a, float4* b, size_t n4, int reps) {
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
      float4 x = a[i]; x.x += 1.f; b[i] = x;
    }
}

int main(int argc, char** argv) {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  const size_t pb = argc > 1 ? atoll(argv[1]) : 76094464;
  printf("devices %d payload %zu\n", ndev, pb);
  for (int policy = 0; policy < 3; ++policy) {
    std::vector<ncclComm_t> comms(ndev);
    std::vector<int> devs(ndev);
    for (int i = 0; i < ndev; ++i) devs[i] = i;
    ncclUniqueId id;
    NK(ncclGetUniqueId(&id));
    NK(ncclGroupStart());
    for (int i = 0; i < ndev; ++i) {
      CK(cudaSetDevice(i));
      ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
      if (policy == 2) cfg.CTAPolicy = NCCL_CTA_POLICY_ZERO;
      if (policy == 1) cfg.maxCTAs = 4;
      NK(ncclCommInitRankConfig(&comms[i], ndev, id, i, &cfg));
    }
    NK(ncclGroupEnd());
    std::vector<void*> buf(ndev);
    std::vector<ncclWindow_t> win(ndev);
    std::vector<cudaStream_t> cs(ndev), ks(ndev);
    std::vector<float*> sa(ndev), sb(ndev);
    const size_t n4 = (size_t)1 << 26;  // 1 GiB per array
    for (int i = 0; i < ndev; ++i) {
      CK(cudaSetDevice(i));
      if (policy == 2) NK(ncclMemAlloc(&buf[i], pb * ndev));
      else CK(cudaMalloc(&buf[i], pb * ndev));
      CK(cudaStreamCreateWithFlags(&cs[i], cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&ks[i], cudaStreamNonBlocking));
      CK(cudaMalloc(&sa[i], n4 * 16));
      CK(cudaMalloc(&sb[i], n4 * 16));
    }
    if (policy == 2) {
      NK(ncclGroupStart());
      for (int i = 0; i < ndev; ++i) {
        CK(cudaSetDevice(i));
        NK(ncclCommWindowRegister(comms[i], buf[i], pb * ndev, &win[i], NCCL_WIN_COLL_SYMMETRIC));
      }
      NK(ncclGroupEnd());
    }
    for (int mode = 0; mode < 2; ++mode) {  // 0: gather alone, 1: with a streaming kernel on every GPU
      std::vector<cudaEvent_t> e0(ndev), e1(ndev), k0(ndev), k1(ndev);
      for (int it = 0; it < 6; ++it) {
        for (int i = 0; i < ndev; ++i) {
          CK(cudaSetDevice(i));
          CK(cudaEventCreate(&e0[i])); CK(cudaEventCreate(&e1[i])); CK(cudaEventCreate(&k0[i])); CK(cudaEventCreate(&k1[i]));
          CK(cudaDeviceSynchronize());
          if (mode == 1) {
            CK(cudaEventRecord(k0[i], ks[i]));
            stream_kernel<<<148 * 4, 256, 0, ks[i]>>>((const float4*)sa[i], (float4*)sb[i], n4, 1);
            CK(cudaEventRecord(k1[i], ks[i]));
          }
          CK(cudaEventRecord(e0[i], cs[i]));
        }
        NK(ncclGroupStart());
        for (int i = 0; i < ndev; ++i) {
          CK(cudaSetDevice(i));
          NK(ncclAllGather((char*)buf[i] + i * pb, buf[i], pb, ncclUint8, comms[i], cs[i]));
        }
        NK(ncclGroupEnd());
        for (int i = 0; i < ndev; ++i) { CK(cudaSetDevice(i)); CK(cudaEventRecord(e1[i], cs[i])); }
        for (int i = 0; i < ndev; ++i) { CK(cudaSetDevice(i)); CK(cudaDeviceSynchronize()); }
        if (it >= 3) {
          float g = 0, k = 0;
          CK(cudaEventElapsedTime(&g, e0[0], e1[0]));
          if (mode == 1) CK(cudaEventElapsedTime(&k, k0[0], k1[0]));
          printf("policy %s mode %s: gather %.3f ms (%.0f GB/s ingress)  stream kernel %.3f ms\n",
                 policy == 0 ? "default" : policy == 1 ? "maxCTAs4" : "ZERO+symm", mode ? "contended" : "alone", g,
                 (ndev - 1) * pb / (g * 1e6), k);
        }
      }
    }
    // kernel alone for reference
    {
      cudaEvent_t a, b; CK(cudaSetDevice(0)); CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
      CK(cudaEventRecord(a, ks[0]));
      stream_kernel<<<148 * 4, 256, 0, ks[0]>>>((const float4*)sa[0], (float4*)sb[0], n4, 1);
      CK(cudaEventRecord(b, ks[0])); CK(cudaDeviceSynchronize());
      float k; CK(cudaEventElapsedTime(&k, a, b)); printf("stream kernel alone %.3f ms\n", k);
    }
    for (int i = 0; i < ndev; ++i) {
      CK(cudaSetDevice(i));
      if (policy == 2) { NK(ncclCommWindowDeregister(comms[i], win[i])); NK(ncclMemFree(buf[i])); }
      else CK(cudaFree(buf[i]));
      CK(cudaFree(sa[i])); CK(cudaFree(sb[i]));
      NK(ncclCommDestroy(comms[i]));
    }
  }
  return 0;
}
