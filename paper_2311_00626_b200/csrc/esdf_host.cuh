// Host-side ESDF helpers shared by esdf.cu (single map) and shard.cu (sharded).
#pragma once

#include "esdf_lower.cuh"

namespace vxm {

// Scratch layout for one ESDF call (ctx->tmp[...]).
struct EsdfScratch {
  uint64_t* merged;
  uint64_t* eff_keys;
  int32_t* eff_tslot;
  int32_t* eff_eslot;
  uint64_t* new_keys;
  int32_t* new_slots;
  uint8_t* flags;
  uint32_t* counts;  // [0] n_eff, [1] n_new, [2] n_old, [3] n_out, [4..] misc
};

Limits limits_for(const vxm_esdf_config& cfg, double vs);
uint32_t grid_for(Context* ctx, uint64_t n, int per_sm = 8);
EsdfScratch esdf_scratch(Context* ctx, uint32_t n_upd_cap, uint32_t n_all_cap);
// effective set + ESDF allocation + neighbour table + sorted-set merge + mark
uint32_t esdf_mark_phase(Layer* E, Layer* T, BlockList* updated, const vxm_esdf_config& cfg,
                         EsdfScratch& s, uint32_t epoch, bool mark_skip = false);
LowerArgs lower_args(Layer* E, const vxm_esdf_config& cfg);
void launch_compact_keys(Context* ctx, const uint64_t* in, const uint8_t* flags,
                         const uint32_t* n_ptr, uint32_t n_cap, uint64_t* out, uint32_t* n_out,
                         const DevStatus* guard, const char* prof_name);

}  // namespace vxm
