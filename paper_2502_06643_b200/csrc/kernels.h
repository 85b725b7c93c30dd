// kernels.h -- host-side launch entry points of the libmoe kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace moe {

// K1 / K9 (route.cu)
void launch_route(const float* logits, int T, int E, int k, int32_t* idx, float* w, cudaStream_t s);
void launch_route_stats(const int32_t* idx_l, const int32_t* idx_l1, int T, int E, int k, int64_t* load,
                        int64_t* coact, int* err, int num_sms, cudaStream_t s);

// Dispatch plan arguments shared by K2/K3/K8 (dispatch.cu).
struct PlanArgs {
  int T;        // tokens of this process in this call
  int k;
  int E;
  int H;
  int V;        // sources handled by this process (1 real, G virtual)
  int G;        // EP group size
  int me;       // real rank (0 in virtual mode)
  int virt;     // 1 = virtual ranks (every expert hosted by this process)
  int n_tiles;  // sum over sources of ceil(T_s / kTileTokens)
};

// Device-side plan state (all int32, allocated by the context).
struct PlanBuffers {
  const int32_t* P;    // [E] placement
  int32_t* tile_hist;  // [n_tiles][E]
  int32_t* tile_base;  // [n_tiles][E]  within-source exclusive prefix
  int32_t* cnt_local;  // [V][E]
  const int32_t* cnt_all;  // [G][E]
  int32_t* base_row;   // [V][E]
  int32_t* seg_meta;   // [1 + 3E + 4]: nseg, seg_row0[E], seg_rows[E], seg_w[E], totals
  int32_t* row_of_item;  // [T*k]: row >= 0 local, -(row+2) remote, -1 invalid
  int* err;
};

int plan_tiles(int T, int V);
void launch_count(const PlanArgs& a, const int32_t* idx, const PlanBuffers& b, cudaStream_t s);
void launch_scan(const PlanArgs& a, const PlanBuffers& b, cudaStream_t s);
void launch_layout(const PlanArgs& a, const PlanBuffers& b, int64_t cap_rows, cudaStream_t s);
void launch_scatter(const PlanArgs& a, const uint16_t* x, const int32_t* idx, const PlanBuffers& b,
                    uint16_t* recv, uint16_t* sendbuf, cudaStream_t s);
void launch_combine(const PlanArgs& a, const float* w, const PlanBuffers& b, const uint16_t* ybuf,
                    const uint16_t* retbuf, uint16_t* out, cudaStream_t s);
void launch_pack_w13(const uint16_t* w1, const uint16_t* w3, int n, int F, int H, uint16_t* w13,
                     cudaStream_t s);

// K5/K6 grouped GEMM (gemm.cu).
struct GemmPlan;  // opaque
int gemm_block_n(int N, bool swiglu);
int gemm_b_box_rows(int N, bool swiglu);  // TMA box rows of the B (weight) operand per CTA
int pack_block(int F);
// Launch the persistent grouped GEMM: D[rows][ldd] for every hosted expert segment.
// tmA / tmB are CUtensorMap (128 bytes each) built by make_tmap_2d.
cudaError_t launch_grouped_gemm(const void* tmA, const void* tmB, uint16_t* D, int ldd, const int32_t* seg_meta,
                                int E, int N, int K, bool swiglu, int num_sms, cudaStream_t s);
// Encode a 2D bf16 K-major tensor map [rows][cols] with box {64, box_rows}, 128B swizzle.
bool make_tmap_2d(void* tmap_out, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows);

}  // namespace moe
