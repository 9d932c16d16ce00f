// plan.cuh — device workspace shared by route -> permute -> expert FFN kernels.
#pragma once
#include <stdint.h>
#include <vector_types.h>

namespace moqe_gpu {

constexpr int kGemvMaxRows = 12;   // experts with <= this many routed rows take the GEMV path (2 passes)

// All pointers are device memory owned by the bank's workspace.
struct Plan {
    int32_t* expert;      // [T*k]  routed expert per (token, slot)
    float* gate;          // [T*k]  gate per (token, slot)
    int32_t* lrank;       // [T*k]  stable rank among same-expert rows inside its route CTA
    int32_t* cta_counts;  // [n_route_ctas * E] per-CTA histogram -> per-CTA base after plan
    int32_t* counts;      // [E]
    int32_t* offsets;     // [E+1] exclusive scan of counts
    int32_t* perm_token;  // [T*k]  token of permuted row pos (rows grouped by expert, ascending token)
    float* perm_gate;     // [T*k]
    int32_t* inv_pos;     // [T*k]  permuted row of (token, slot)
    int32_t* gemv_list;   // [E]    experts for the GEMV path (expert order)
    int32_t* gemm_list;   // [E]    experts for the tcgen05 path
    int32_t* gemm_tile_start;  // [E+1] prefix of GEMM tiles per listed expert (per m-tile row)
    int32_t* meta;        // [8]    0: n_gemv, 1: n_gemm, 2: gemm n-tiles total, 3: max n_e, 5: forward epoch
    unsigned* tickets;    // [8]    0: route last-CTA, 1: gemv fc1 items, 2: gemm fc1, 3: gemm fc2, 4: gemv fc2
    unsigned* done;       // [E]    (reserved; reset per forward)
    float* logits;        // [T][E] router logits (large-T path)
    int4* gtab;           // [E+1] GEMV table: [0].x = n_gemv, [1+a] = {expert, rows, row offset, 0} (one load round)
};

}  // namespace moqe_gpu
