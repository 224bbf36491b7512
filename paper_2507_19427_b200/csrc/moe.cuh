// moe.cuh — argument blocks of the MoE FFN kernels (K5-K9).
#pragma once
#include <cuda_bf16.h>

#include <cstdint>

namespace afdk {
namespace moe {

constexpr int kMaxExperts = 64;  // routed experts (Step-3: 48)
constexpr int kMaxTopK = 8;      // Step-3: 3
constexpr int kChunk = 64;       // dispatched rows per GEMM work item (MMA N <= 64)
constexpr int kChunkMX = 128;    // rows per work item of the MXFP8 (block-scaled MMA) GEMMs
constexpr int kChunkMX2 = 256;   // rows per work item of the CTA-pair MXFP8 GEMMs
constexpr int kChunkMX2Two = 384;  // ... in their two-accumulator form

struct RouterArgs {
  const __nv_bfloat16* h;       // [T, H] post-attention RMSNorm output
  const __nv_bfloat16* gate_w;  // [E, H]
  int T, H, E, k, renormalize;
  float* logits;                // [T, E] optional
  int32_t* ids;                 // [T, k]
  float* weights;               // [T, k]
  uint8_t* xq;                  // [T, H] e4m3, optional (dispatch payload)
  float* xs;                    // [T, H/128]
};

struct Work {
  int group;  // expert id, or E for the shared expert
  int row0;   // first row of this item in the intermediate / output buffers
  int rows;   // <= chunk
  int xrow0;  // first row of its W13 input (MoE: = row0 in the dispatch buffer;
              // dense FFN splits: the token row, shared by every split)
  int gfirst, gcnt;  // its group's chunks: work[gfirst, gfirst + gcnt)
};

// GEMM item order over (group, m-tile, chunk): a group's chunks are adjacent,
// so they share each weight tile while it is in L2, and a chunk's activation
// panel is re-read by the group's m-tiles within one wave.  Items of a group
// occupy [gfirst*m_tiles, (gfirst+gcnt)*m_tiles), hence any chunk index
// it/m_tiles inside that range names the group.
struct ItemRef {
  int mt, chunk;
};
__device__ __forceinline__ ItemRef item_of(const Work* work, int it, int m_tiles) {
  const Work w = work[it / m_tiles];
  const int local = it - w.gfirst * m_tiles;
  return {local / w.gcnt, w.gfirst + local % w.gcnt};
}

struct PermuteArgs {
  const int32_t* ids;  // [T, k]
  int T, k, E;
  int expert_lo, expert_hi;        // routed experts owned by this FFN rank
  int shared_local, shared_lo, shared_hi;  // shared-expert token range owned here
  int32_t* offsets;    // [E+1]
  int32_t* perm;       // [T*k] slot -> t*k+j
  int32_t* inv;        // [T*k] t*k+j -> slot
  Work* work;          // [max work]
  int* n_work;
  int chunk;           // rows per work item (kChunk or kChunkMX)
  int* sched = nullptr;  // optional: zeroed [sched_len] (queue head + per-chunk counters of the fused kernel)
  int sched_len = 0;
};

struct GatherArgs {
  const uint8_t* xq;   // [T, H]
  const float* xs;     // [T, H/128]
  const int32_t* perm;
  int T, k, H, rows_pad;
  uint8_t* xp;         // [rows_pad, H]  routed rows then shared rows
  float* xs_t;         // [H/128, rows_pad]
  const uint8_t* xsf;  // MXFP8 mode (xs == nullptr): [T, H/32] UE8M0 scales
  uint8_t* xsf_p;      //   gathered [rows_pad, H/32]
};

struct CombineArgs {
  const float* y;      // [rows_pad, H] expert outputs in dispatch order
  const int32_t* ids;
  const float* weights;
  const int32_t* inv;
  int T, k, H;
  int expert_lo, expert_hi, shared_local, shared_lo, shared_hi;
  __nv_bfloat16* out;  // [T, H]
  // fused F->A return (optional): token row t goes to
  // dst[t / rows_per_dst] + (t % rows_per_dst) * H (peer memory over NVLink)
  const uint64_t* dst;
  int rows_per_dst;
};

inline int max_work(int T, int k, int E) { return E + (T * k) / kChunk + 1 + T / kChunk + 1; }
inline int rows_pad(int T, int k) { return ((T * k + T + 127) / 128) * 128; }
// MX work items read a full 128-row panel (scale rows by plain loads): keep
// one spare panel so the last chunk never runs off the buffer
inline int rows_pad_mx(int T, int k) { return rows_pad(T, k) + kChunkMX; }

struct QuantMxArgs {
  const __nv_bfloat16* x;  // [T, H]
  int T, H;
  uint8_t* q;              // [T, H] e4m3
  uint8_t* sf;             // [T, H/32] UE8M0
};

}  // namespace moe
}  // namespace afdk
