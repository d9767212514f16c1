// nvls_probe.cu — probe: NCCL device API multicast (NVLS) stores into a
// symmetric window.  Every rank multimem-stores its rank id into word `rank`
// of a small region; every rank then checks it sees all ids.  Also times a
// unicast vs multicast push of one 76 MB payload.  Single process, all GPUs.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
#define NK(x) do { ncclResult_t r = (x); if (r != ncclSuccess) { printf("NCCL %s @%d\n", ncclGetErrorString(r), __LINE__); exit(1);} } while (0)

__global__ void k_mc_ids(ncclWindow_t w, ncclMultimemHandle mm, int rank) {
  unsigned* p = (unsigned*)ncclGetMultimemPointer(w, 4 * rank, mm);
  asm volatile("multimem.st.global.u32 [%0], %1;" ::"l"(p), "r"((unsigned)(100 + rank)) : "memory");
}

__global__ void k_push(ncclWindow_t w, ncclMultimemHandle mm, int rank, int M, size_t pb, int mc) {
  const size_t nw = pb / 4;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nw; i += (size_t)gridDim.x * blockDim.x) {
    const size_t off = rank * pb + 4 * i;
    const unsigned v = (unsigned)i;
    if (mc) {
      unsigned* p = (unsigned*)ncclGetMultimemPointer(w, off, mm);
      asm volatile("multimem.st.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
    } else {
      for (int q = 0; q < M; ++q) *(unsigned*)ncclGetLsaPointer(w, off, q) = v;
    }
  }
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
  for (int i = 0; i < ndev; ++i) printf("rank %d mcBasePtr %p\n", i, dc[i].lsaMultimem.mcBasePtr);
  std::vector<void*> buf(ndev);
  std::vector<ncclWindow_t> win(ndev);
  const size_t bytes = ((pb * ndev + (2 << 20) - 1) / (2 << 20)) * (2 << 20);
  for (int i = 0; i < ndev; ++i) {
    CK(cudaSetDevice(i));
    NK(ncclMemAlloc(&buf[i], bytes));
    CK(cudaMemset(buf[i], 0, bytes));
  }
  NK(ncclGroupStart());
  for (int i = 0; i < ndev; ++i) {
    CK(cudaSetDevice(i));
    NK(ncclCommWindowRegister(comms[i], buf[i], bytes, &win[i], NCCL_WIN_COLL_SYMMETRIC));
  }
  NK(ncclGroupEnd());
  for (int i = 0; i < ndev; ++i) { CK(cudaSetDevice(i)); CK(cudaDeviceSynchronize()); }
  if (dc[0].lsaMultimem.mcBasePtr == nullptr) { printf("no multimem\n"); return 0; }
  for (int i = 0; i < ndev; ++i) {
    CK(cudaSetDevice(i));
    k_mc_ids<<<1, 1>>>(win[i], dc[i].lsaMultimem, i);
  }
  for (int i = 0; i < ndev; ++i) { CK(cudaSetDevice(i)); CK(cudaDeviceSynchronize()); }
  for (int i = 0; i < ndev; ++i) {
    CK(cudaSetDevice(i));
    std::vector<unsigned> h(ndev);
    CK(cudaMemcpy(h.data(), buf[i], 4 * ndev, cudaMemcpyDeviceToHost));
    printf("rank %d sees:", i);
    for (int q = 0; q < ndev; ++q) printf(" %u", h[q]);
    printf("\n");
  }
  for (int mc = 0; mc < 2; ++mc) {
    for (int it = 0; it < 4; ++it) {
      std::vector<cudaEvent_t> e0(ndev), e1(ndev);
      for (int i = 0; i < ndev; ++i) {
        CK(cudaSetDevice(i));
        CK(cudaEventCreate(&e0[i])); CK(cudaEventCreate(&e1[i]));
        CK(cudaEventRecord(e0[i]));
        k_push<<<148 * 8, 256>>>(win[i], dc[i].lsaMultimem, i, ndev, pb, mc);
        CK(cudaEventRecord(e1[i]));
      }
      for (int i = 0; i < ndev; ++i) { CK(cudaSetDevice(i)); CK(cudaDeviceSynchronize()); }
      float ms; CK(cudaEventElapsedTime(&ms, e0[0], e1[0]));
      if (it >= 2) printf("%s push of %zu bytes to %d ranks: %.3f ms (ingress %.0f GB/s)\n", mc ? "multicast" : "unicast", pb, ndev, ms, (ndev - 1) * pb / (ms * 1e6));
    }
  }
  // verify the last push: every rank holds word i = i in every slot
  for (int i = 0; i < ndev; ++i) {
    CK(cudaSetDevice(i));
    std::vector<unsigned> h(pb / 4);
    int bad = 0;
    for (int q = 0; q < ndev; ++q) {
      CK(cudaMemcpy(h.data(), (char*)buf[i] + q * pb, pb, cudaMemcpyDeviceToHost));
      for (size_t k = 0; k < pb / 4; k += 4099) bad += h[k] != (unsigned)k;
    }
    printf("rank %d push check: %s\n", i, bad ? "BAD" : "ok");
  }
  return 0;
}
