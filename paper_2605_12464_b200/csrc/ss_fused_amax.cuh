// ss_fused_amax.cuh — the amax warps of the fused-amax quantize kernel
// (quant_kernel<..., AF>): step a2 (tensor amax) for a batch, run by
// kAmaxWarps warps per CTA ahead of the search.
//
// Units of kAmaxUnitVecs 16-B vectors of the amax tasks (QuantBatch::am) are
// drawn in order from one counter (QuantBatch::done[kMaxTensors]).  Each
// unit's max of |x| is folded into its task's slot (atomicMax of the FP32 bit
// pattern; exact, and non-finite inputs sort above every finite value, R14),
// then done[i] is release-incremented; search warps acquire done[i] == na
// before using G.  The tasks are the launch's own tensors (per-tensor G on
// one GPU), or the NEXT group's shards of a sharded step, whose local amaxes
// then go to the all-reduce while this launch searches
// (ss_quantize_nvfp4_batched_next_amax).
// Reductions use HMNMX2 (max.NaN.xorsign.abs.bf16x2): the magnitude max of
// bf16 pairs with NaN propagation in one instruction; the sign bits it leaves
// are masked off once per unit.
#pragma once
#include "ss_search.cuh"

namespace ss {

// max(|a|, |b|) per bf16 lane (NaN-propagating; sign bit = xor, masked later)
__device__ __forceinline__ uint32_t hmax_abs2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.NaN.xorsign.abs.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t hmax_abs_vec(uint32_t m, const uint4& a) {
  return hmax_abs2(m, hmax_abs2(hmax_abs2(a.x, a.y), hmax_abs2(a.z, a.w)));
}

// Fold a unit's per-lane magnitude maxima into task ta's amax, then count the unit.
// Peer-memory exchange, producer side: `count` local amaxes
// are complete; one warp stores them into every rank's exchange buffer
// (lanes stride tensors x ranks), makes the stores visible system-wide, then
// releases each rank's flag word for this rank with `epoch`.
__device__ __forceinline__ void exchange_store(const uint32_t* local, int count, int world, uint32_t epoch,
                                               uint32_t* const* slots, uint32_t* const* flags, int lane) {
  const int n = count * world;
  for (int k = lane; k < n; k += 32) {
    const int j = k / world, r = k - j * world;
    st_relaxed_sys(slots[r] + j * kMaxPeers, ld_relaxed_gpu(local + j));
  }
  __threadfence_system();
  __syncwarp();
  if (lane < world) st_release_sys(flags[lane], epoch);
}
__device__ __forceinline__ void exchange_out(const QuantBatch& p, int lane) {
  exchange_store(p.xlocal, p.xcount_out, p.xw, p.xepoch_out, p.xout, p.xout_flag, lane);
}

// The same from its own one-warp launch, after a separate amax pass (stream order).
struct XPub {
  const uint32_t* local;
  int count, world;
  uint32_t epoch;
  uint32_t* slots[kMaxPeers];
  uint32_t* flags[kMaxPeers];
};
__global__ void __launch_bounds__(32) exchange_publish_kernel(const __grid_constant__ XPub x) {
  exchange_store(x.local, x.count, x.world, x.epoch, x.slots, x.flags, threadIdx.x);
}

__device__ __forceinline__ void amax_publish(const QuantBatch& p, int ta, uint32_t m, int lane) {
  m &= 0x7FFF7FFFu;
  const uint32_t r = __reduce_max_sync(0xFFFFFFFFu, max(m & 0xFFFFu, m >> 16));
  uint32_t last = 0;
  if (lane == 0) {
    const AmaxTask& A = p.am[ta];
    if (r && (r << 16) > ld_relaxed_gpu(A.slot)) atomicMax(A.slot, r << 16);
    if (A.done >= 0) {
      red_release_add_gpu(p.done + A.done, 1u);
    } else if (p.xunits_out > 0) {  // a next-group unit of an exchanging launch
      last = atom_add_acq_rel_gpu(p.done + kMaxTensors + 1, 1u) == (uint32_t)p.xunits_out - 1;
    }
  }
  if (__shfl_sync(0xFFFFFFFFu, last, 0)) exchange_out(p, lane);  // warp-uniform
}

__device__ __forceinline__ uint32_t amax_draw(const QuantBatch& p, int lane) {
  uint32_t idx = 0;
  if (lane == 0) idx = atomicAdd(p.done + kMaxTensors, 1u);
  return __shfl_sync(0xFFFFFFFFu, idx, 0);
}

// Unit u -> its task (forward walk from `t`) and 16-B vector range [v0, v1).
__device__ __forceinline__ void amax_unit(const QuantBatch& p, uint32_t u, int& t, int64_t& v0, int64_t& v1) {
  const int ns = p.ntrail ? p.tr0 : p.nam;  // trail tasks (numbered apart) follow
  while (t + 1 < ns && p.am[t + 1].a0 <= (int)u) t++;
  const AmaxTask& A = p.am[t];
  v0 = (int64_t)((int)u - A.a0) * kAmaxUnitVecs;
  v1 = min(A.nvec, v0 + kAmaxUnitVecs);
}

// Trailing amax (QuantBatch::ntrail).
// Publish a warp's per-lane running max m (bf16 |x| pairs) into task t's slot:
// atomicMax of the FP32 bits, fire-and-forget; NaN sorts above every finite
// value as in amax_publish (R14).
__device__ __forceinline__ void trail_publish(const QuantBatch& p, int t, uint32_t m, int lane) {
  m &= 0x7FFF7FFFu;
  const uint32_t r = __reduce_max_sync(0xFFFFFFFFu, max(m & 0xFFFFu, m >> 16));
  if (lane == 0 && r) atomicMax(p.am[t].slot, r << 16);
}
// Fold the trail units of scheduling unit su into their tensors' amax slots
// (the whole warp: 8 coalesced 16-B loads per lane per 4-KiB unit, HMNMX2; one
// publish per tensor the units touch).  A full unit loads from one base
// address with constant offsets; only a tensor's last unit is predicated.
// The loads are not prefetched: an L2 prefetch one work item ahead (per-lane
// prefetch.global.L2 or a bulk prefetch) measured slower (C2 r = 8: 14.53 vs
// 14.32 ms per step).
__device__ __forceinline__ void trail_fold(const QuantBatch& p, int64_t su, int& t, int lane) {
  if (su * p.tpu >= p.ntrail) return;  // (also keeps u0 within 32 bits)
  const int u0 = (int)(su * p.tpu);
  const int ue = min(u0 + p.tpu, p.ntrail);
  uint32_t m = 0;
  for (int u = u0; u < ue; u++) {
    int tn = t < p.tr0 ? p.tr0 : t;
    while (tn + 1 < p.nam && p.am[tn + 1].a0 <= u) tn++;
    if (tn != t) {  // warp-uniform
      if (t >= p.tr0) trail_publish(p, t, m, lane);
      m = 0;
      t = tn;
    }
    const AmaxTask& A = p.am[t];
    const int64_t v0 = (int64_t)(u - A.a0) * kTrailVecs;
    const uint4* src = A.in + v0 + lane;
    const int64_t left = A.nvec - v0;
    if (left >= kTrailVecs) {  // warp-uniform
      uint4 a[kTrailVecs / 32];
#pragma unroll
      for (int jj = 0; jj < kTrailVecs / 32; jj++) a[jj] = __ldcs(src + 32 * jj);
#pragma unroll
      for (int jj = 0; jj < kTrailVecs / 32; jj++) m = hmax_abs_vec(m, a[jj]);
    } else {
      const int n = (int)left;
#pragma unroll
      for (int jj = 0; jj < kTrailVecs / 32; jj++)
        if (lane + 32 * jj < n) m = hmax_abs_vec(m, __ldcs(src + 32 * jj));
    }
  }
  if (t >= p.tr0 && ue > u0) trail_publish(p, t, m, lane);
}

// One amax warp: kAmaxWarpVecs coalesced 16-B loads in flight per lane; the next unit is
// drawn one ahead and bulk-prefetched into L2 (TMA, no registers or shared
// memory), so these loads mostly hit L2.  (Staging the units through
// shared memory with TMA bulk copies instead was measured slower: 2.4 vs
// 1.5 ms for the amax of 6.9 G elements under the search.)
__device__ __forceinline__ void amax_warp(const QuantBatch& p, int lane) {
  int ta = 0, tn = 0;
  auto prefetch = [&](uint32_t u) {
    int64_t v0, v1;
    amax_unit(p, u, tn, v0, v1);
    if (lane == 0) prefetch_l2_bulk(p.am[tn].in + v0, (uint32_t)(16 * (v1 - v0)));
  };
  uint32_t nxt = amax_draw(p, lane);
  if (nxt < (uint32_t)p.namax) prefetch(nxt);
  while (nxt < (uint32_t)p.namax) {
    const uint32_t idx = nxt;
    nxt = amax_draw(p, lane);
    if (nxt < (uint32_t)p.namax) prefetch(nxt);
    int64_t v0, v1;
    amax_unit(p, idx, ta, v0, v1);
    const uint4* src = p.am[ta].in;
    uint32_t m = 0;
    for (int64_t v = v0 + lane; v < v1; v += 32 * kAmaxWarpVecs) {
      uint4 a[kAmaxWarpVecs];
#pragma unroll
      for (int k = 0; k < kAmaxWarpVecs; k++)
        a[k] = v + 32 * k < v1 ? __ldcs(src + v + 32 * k) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
      for (int k = 0; k < kAmaxWarpVecs; k++) m = hmax_abs_vec(m, a[k]);
    }
    amax_publish(p, ta, m, lane);
  }
}

}  // namespace ss
