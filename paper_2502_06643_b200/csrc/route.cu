// route.cu -- K1 fused softmax+top-k gating and K9 routing-statistics counting.
//
// K1 implements moe_route ("top-2 router ... two most relevant
// experts"; Mixtral gate = softmax over the top-k logits, reading G1), with the
// tie rule of reading G2: descending logit, ties to the lower expert id,
// -0.0 == +0.0.
// K9 implements moe_route_stats: P_{e,l} and R_{e1,e2,l} with
// k x k pairs per token (reading G10).
#include "common.cuh"
#include "kernels.h"

namespace moe {

// Order-preserving map float -> uint32 (larger float -> larger key).
__device__ __forceinline__ uint32_t ordered_key(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_to_float(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  return __uint_as_float(u);
}

// LPT lanes cooperate on one token; each lane holds VPL logits (e = lane + v*LPT).
// k rounds of a packed 64-bit max-reduction over (ordered logit, ~e): the
// winner of a round is the largest remaining logit, ties to the lower id.
template <int LPT, int VPL>
__global__ void __launch_bounds__(256) k_route(const float* __restrict__ logits, int T, int E, int k,
                                               int32_t* __restrict__ idx, float* __restrict__ w, int* err) {
  constexpr int TPW = 32 / LPT;  // tokens per warp
  const int lane = threadIdx.x & 31;
  const int gl = lane % LPT;
  const long long warp = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const long long t = warp * TPW + lane / LPT;
  const bool valid = t < T;

  uint64_t key[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int e = gl + v * LPT;
    if (valid && e < E) {
      float l = __ldg(logits + t * E + e) + 0.0f;  // -0.0 -> +0.0
      if (l != l) atomicOr(err, kErrNaN);           // NaN: the selection is undefined
      key[v] = ((uint64_t)ordered_key(l) << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)e);
    } else {
      key[v] = 0;  // below every real key
    }
  }

  float l0 = 0.f, sum = 0.f, my_l = 0.f;
  int my_e = 0;
  for (int r = 0; r < k; ++r) {
    uint64_t best = 0;
#pragma unroll
    for (int v = 0; v < VPL; ++v) best = key[v] > best ? key[v] : best;
#pragma unroll
    for (int off = LPT / 2; off > 0; off >>= 1) {
      uint64_t o = __shfl_xor_sync(0xffffffffu, best, off, LPT);
      best = o > best ? o : best;
    }
    const int e = (int)(0xFFFFFFFFu - (uint32_t)(best & 0xFFFFFFFFu));
    const float l = key_to_float((uint32_t)(best >> 32));
    if (r == 0) l0 = l;
    sum += expf(l - l0);
#pragma unroll
    for (int v = 0; v < VPL; ++v)
      if (key[v] == best) key[v] = 0;  // remove the winner (only its owner matches)
    if (gl == r) {
      my_e = e;
      my_l = l;
    }
  }
  if (valid && gl < k) {
    idx[t * k + gl] = my_e;
    w[t * k + gl] = expf(my_l - l0) / sum;
  }
}

void launch_route(const float* logits, int T, int E, int k, int32_t* idx, float* w, int* err, cudaStream_t s) {
  if (T <= 0) return;
  const int threads = 256;
  auto go = [&](auto kern, int lpt) {
    long long tokens_per_block = (threads / 32) * (32 / lpt);
    int blocks = (int)((T + tokens_per_block - 1) / tokens_per_block);
    kern<<<blocks, threads, 0, s>>>(logits, T, E, k, idx, w, err);
  };
  if (E <= 4) go(k_route<4, 1>, 4);
  else if (E <= 8) go(k_route<8, 1>, 8);
  else if (E <= 16) go(k_route<16, 1>, 16);
  else if (E <= 32) go(k_route<32, 1>, 32);
  else if (E <= 64) go(k_route<32, 2>, 32);
  else if (E <= 128) go(k_route<32, 4>, 32);
  else go(k_route<32, 8>, 32);
}

// ------------------------------------------------------------------------ K9
// Shared-memory histograms (load [E], coact [E][E]) with warp-aggregated
// increments (__match_any_sync), flushed to int64 global counters.  For E > 128
// the E x E co-activation histogram does not fit in shared memory: its
// (warp-aggregated) increments go straight to the int64 global counters.
__global__ void __launch_bounds__(256) k_route_stats(const int32_t* __restrict__ idx_l,
                                                     const int32_t* __restrict__ idx_l1, int T, int E, int k,
                                                     unsigned long long* __restrict__ load,
                                                     unsigned long long* __restrict__ coact, int* err,
                                                     int smem_co) {
  extern __shared__ int hist[];  // [E] load, then [E*E] coact (smem_co)
  int* hload = hist;
  int* hco = hist + E;
  const int nbins = E + (idx_l1 && smem_co ? E * E : 0);
  for (int b = threadIdx.x; b < nbins; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (long long base = (long long)blockIdx.x * blockDim.x; base < T; base += (long long)gridDim.x * blockDim.x) {
    const long long t = base + threadIdx.x;
    const bool valid = t < T;
    for (int j1 = 0; j1 < k; ++j1) {
      int e1 = valid ? idx_l[t * k + j1] : -1;
      if (valid && (e1 < 0 || e1 >= E)) {
        atomicOr(err, kErrBadExpert);
        e1 = -1;
      }
      unsigned m = __match_any_sync(0xffffffffu, e1);
      if (e1 >= 0 && lane == __ffs(m) - 1) atomicAdd(&hload[e1], __popc(m));
      if (idx_l1) {
        for (int j2 = 0; j2 < k; ++j2) {
          int e2 = valid ? idx_l1[t * k + j2] : -1;
          if (valid && (e2 < 0 || e2 >= E)) {
            atomicOr(err, kErrBadExpert);
            e2 = -1;
          }
          int bin = (e1 >= 0 && e2 >= 0) ? e1 * E + e2 : -1;
          unsigned m2 = __match_any_sync(0xffffffffu, bin);
          if (bin >= 0 && lane == __ffs(m2) - 1) {
            if (smem_co) atomicAdd(&hco[bin], __popc(m2));
            else atomicAdd(&coact[bin], (unsigned long long)__popc(m2));
          }
        }
      }
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nbins; b += blockDim.x) {
    int v = hist[b];
    if (v) {
      if (b < E) atomicAdd(&load[b], (unsigned long long)v);
      else atomicAdd(&coact[b - E], (unsigned long long)v);
    }
  }
}

void launch_route_stats(const int32_t* idx_l, const int32_t* idx_l1, int T, int E, int k, int64_t* load,
                        int64_t* coact, int* err, int num_sms, cudaStream_t s) {
  if (T <= 0) return;
  const int threads = 256;
  int blocks = (T + threads - 1) / threads;
  if (blocks > 2 * num_sms) blocks = 2 * num_sms;
  const int smem_co = E <= 128 ? 1 : 0;
  size_t smem = sizeof(int) * (E + (idx_l1 && smem_co ? E * E : 0));
  static unsigned long long attr = 0;  // per device
  if (first_time_on_device(attr))  // E up to 128 needs > 48 KB for the E x E histogram
    cudaFuncSetAttribute(k_route_stats, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(int) * (128 + 128 * 128)));
  k_route_stats<<<blocks, threads, smem, s>>>(idx_l, idx_l1, T, E, k, (unsigned long long*)load,
                                              (unsigned long long*)coact, err, smem_co);
}

void preload_route_kernels() {
  cudaFuncAttributes fa;
  const void* fs[] = {(const void*)k_route<4, 1>, (const void*)k_route<8, 1>, (const void*)k_route<16, 1>,
                      (const void*)k_route<32, 1>, (const void*)k_route<32, 2>, (const void*)k_route<32, 4>,
                      (const void*)k_route<32, 8>, (const void*)k_route_stats};
  for (const void* f : fs) cudaFuncGetAttributes(&fa, f);
}

}  // namespace moe
