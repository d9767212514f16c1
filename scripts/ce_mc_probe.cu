// ce_mc_probe.cu — probe: can the copy engines write through an NVLS
// multicast address (one HBM read of the source, NVSwitch replicates to every
// GPU), and is that faster than one peer copy per destination?  Single
// process, all GPUs, one 1B-fragment payload per GPU.  Not part of the product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ce_mc_probe scripts/ce_mc_probe.cu \
//      -I<nccl>/include -L<nccl>/lib -l:libnccl.so.2
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
#define NK(x) do { ncclResult_t r = (x); if (r != ncclSuccess) { printf("NCCL %s @%d\n", ncclGetErrorString(r), __LINE__); exit(1);} } while (0)

__global__ void k_mc_ptr(ncclWindow_t w, ncclMultimemHandle mm, size_t off, void** out) {
  *out = ncclGetMultimemPointer(w, off, mm);
}
__global__ void k_fill(unsigned* p, size_t nw, unsigned tag) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nw; i += (size_t)gridDim.x * blockDim.x)
    p[i] = tag ^ (unsigned)i;
}

int main() {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  const size_t pb = 76094464;
  std::vector<ncclComm_t> comms(ndev);
  ncclUniqueId id;
  NK(ncclGetUniqueId(&id));
  NK(ncclGroupStart());
  for (int i = 0; i < ndev; ++i) {
    CK(cudaSetDevice(i));
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.CTAPolicy = NCCL_CTA_POLICY_ZERO;
    NK(ncclCommInitRankConfig(&comms[i], ndev, id, i, &cfg));
  }
  NK(ncclGroupEnd());
  std::vector<ncclDevComm_t> dc(ndev);
  NK(ncclGroupStart());
  for (int i = 0; i < ndev; ++i) {
    CK(cudaSetDevice(i));
    ncclDevCommRequirements_t req = {};
    req.lsaMultimem = true;
    NK(ncclDevCommCreate(comms[i], &req, &dc[i]));
  }
  NK(ncclGroupEnd());
  const size_t bytes = ((pb * ndev + (2 << 20) - 1) / (2 << 20)) * (2 << 20);
  std::vector<void*> buf(ndev), src(ndev);
  std::vector<ncclWindow_t> win(ndev);
  std::vector<cudaStream_t> st(ndev);
  for (int i = 0; i < ndev; ++i) {
    CK(cudaSetDevice(i));
    NK(ncclMemAlloc(&buf[i], bytes));
    CK(cudaMemset(buf[i], 0, bytes));
    CK(cudaMalloc(&src[i], pb));
    k_fill<<<1184, 256>>>((unsigned*)src[i], pb / 4, 0x1000u * (i + 1));
    CK(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
  }
  NK(ncclGroupStart());
  for (int i = 0; i < ndev; ++i) {
    CK(cudaSetDevice(i));
    NK(ncclCommWindowRegister(comms[i], buf[i], bytes, &win[i], NCCL_WIN_COLL_SYMMETRIC));
  }
  NK(ncclGroupEnd());
  for (int i = 0; i < ndev; ++i) { CK(cudaSetDevice(i)); CK(cudaDeviceSynchronize()); }
  if (dc[0].lsaMultimem.mcBasePtr == nullptr) { printf("no multimem\n"); return 0; }
  std::vector<void*> mc(ndev);
  for (int i = 0; i < ndev; ++i) {
    CK(cudaSetDevice(i));
    void** d;
    CK(cudaMallocManaged(&d, sizeof(void*)));
    k_mc_ptr<<<1, 1>>>(win[i], dc[i].lsaMultimem, (size_t)i * pb, d);
    CK(cudaDeviceSynchronize());
    mc[i] = *d;
    printf("rank %d: multicast address of its slot %p\n", i, mc[i]);
  }
  for (int mode = 0; mode < 2; ++mode) {  // 0: one peer copy per destination, 1: one copy to the multicast address
    for (int it = 0; it < 5; ++it) {
      for (int i = 0; i < ndev; ++i) { CK(cudaSetDevice(i)); CK(cudaMemsetAsync(buf[i], 0, (size_t)ndev * pb, st[i])); CK(cudaStreamSynchronize(st[i])); }
      std::vector<cudaEvent_t> e0(ndev), e1(ndev);
      for (int i = 0; i < ndev; ++i) {
        CK(cudaSetDevice(i));
        CK(cudaEventCreate(&e0[i]));
        CK(cudaEventCreate(&e1[i]));
        CK(cudaEventRecord(e0[i], st[i]));
        if (mode == 0) {
          for (int q = 0; q < ndev; ++q)
            CK(cudaMemcpyPeerAsync((char*)buf[q] + (size_t)i * pb, q, src[i], i, pb, st[i]));
        } else {
          cudaError_t e = cudaMemcpyAsync(mc[i], src[i], pb, cudaMemcpyDeviceToDevice, st[i]);
          if (e != cudaSuccess) { printf("multicast memcpy: %s\n", cudaGetErrorString(e)); return 0; }
        }
        CK(cudaEventRecord(e1[i], st[i]));
      }
      float worst = 0;
      for (int i = 0; i < ndev; ++i) {
        CK(cudaSetDevice(i));
        cudaError_t e = cudaStreamSynchronize(st[i]);
        if (e != cudaSuccess) { printf("mode %d sync: %s\n", mode, cudaGetErrorString(e)); return 0; }
        float ms;
        CK(cudaEventElapsedTime(&ms, e0[i], e1[i]));
        worst = ms > worst ? ms : worst;
      }
      int bad = 0;
      for (int i = 0; i < ndev; ++i) {
        CK(cudaSetDevice(i));
        std::vector<unsigned> h(pb / 4);
        for (int q = 0; q < ndev; ++q) {
          CK(cudaMemcpy(h.data(), (char*)buf[i] + (size_t)q * pb, pb, cudaMemcpyDeviceToHost));
          for (size_t k = 0; k < pb / 4; k += 997) bad += h[k] != ((0x1000u * (q + 1)) ^ (unsigned)k);
        }
      }
      if (it >= 2)
        printf("%s: every GPU's payload to all %d GPUs in %.3f ms (max over GPUs), ingress %.0f GB/s per GPU, %s\n",
               mode ? "multicast CE copy" : "peer CE copies   ", ndev, worst, (ndev - 1) * pb / (worst * 1e6),
               bad ? "DATA WRONG" : "data ok");
    }
  }
  return 0;
}
