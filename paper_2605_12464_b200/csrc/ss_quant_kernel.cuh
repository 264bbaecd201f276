// ss_quant_kernel.cuh — the search-quantize kernel (Algorithm 1 per block, a1 and a3-a7).
#pragma once
#include "ss_fused_amax.cuh"

namespace ss {

// RI: 0 = no per-block row; 1 = the batch needs each block's row (per-row G
// from rowscale_kernel or the swizzled scale layout); 2 = also row-fused
// tensors (their row amax inside this kernel, T.hpr > 0).  Lower levels
// compile the unused steps out.  FMT: block
// format (Fmt<>); fixed windows (NEG >= 0) are compiled for NVFP4 and for
// radius 0..2 of the other formats (ss_api.cu pick_kernel).  Units:
// `b`/`j` index 16-element HALF-blocks (one per lane); a 32-element block is
// the lane pair (2i, 2i + 1), whose even lane writes its scale, offset and
// errors.
//
// AF (fused amax, gmode 1, RI 0): the batch's amax passes (a2) run inside
// this launch.  The last kAmaxWarps warps of every CTA start as amax warps:
// they draw 32-KiB amax units in tensor order from one counter, keep 8
// coalesced 16-B loads in flight per lane, fold each unit's max into the
// tensor's amax slot (atomicMax) and release-increment done[i]; when the
// units run out they join the search.  A search warp waits (acquire) for
// done[i] == na before its first item of tensor i.  The amax warps never
// wait, so the HBM-bound amax runs ahead under the ALU-bound search and no
// schedule can deadlock.  Trailing amax (p.ntrail > 0, §4.2c): the search
// warps also fold the NEXT launch's tensors' amax, a share per scheduling
// unit; nobody in this launch waits for it.
template <int NEG, int POS, int RI, int FMT, bool AF = false>
__global__ void __launch_bounds__(kThreads, SS_MIN_BLOCKS) quant_kernel(const __grid_constant__ QuantBatch p) {
  static_assert(!AF || RI == 0, "fused amax: per-tensor G, plain layout");
  using F = Fmt<FMT>;
  constexpr int Pad = NEG < 0 ? F::kMaxCode : (NEG > POS ? NEG : POS);
  constexpr int TabW = F::SF ? 255 + 2 * Pad : 127 + 2 * Pad;
  constexpr int kHalves = F::BS / 16;  // lanes per scale block
  __shared__ __align__(16) uint4 tab[F::SF ? TabW : 2 * TabW];
  __shared__ __align__(128) uint4 buf[kWarps][kStages][kTaskBytes / 16];

  build_cand_table<Pad, F::SF>(tab);
  __syncthreads();
  // Launched with PDL: everything above overlaps the predecessor (amax /
  // row-scale / previous sums grid); the scheduler counters, amax slots and
  // outputs are touched only after it has completed.
  pdl_wait();
  pdl_launch_dependents();  // the error-sum grid may launch early (it waits for this one)

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gw = blockIdx.x * kWarps + w;

#ifdef SS_AF_TRACE
  auto gtime = []() -> unsigned long long {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
  };
  if (AF && threadIdx.x == 0) atomicMin(p.evals + 0, gtime());
#endif
  if constexpr (AF) {
    if (w >= kWarps - kAmaxWarps) {  // amax warp (a2), then a search warp
      amax_warp(p, lane);
#ifdef SS_AF_TRACE
      if (lane == 0) atomicMax(p.evals + 1, gtime());
#endif
    }
  }

  const float kinv = __uint_as_float(F::kInvVmaxBits);  // RN(1 / vmax) (R8)
  // A work item is up to kTaskBlocks half-blocks of one tensor, named by its
  // tensor and local index li.  Plain tensor: item li covers half-blocks
  // [64 li, 64 li + 64); its items are handed out in scheduling units of
  // p.ipu consecutive items (one ticket and one error-sum partial per unit).
  // Row-fused tensor (T.hpr > 0): item li = r * cpr + c is chunk c of row r,
  // one partial per chunk; its G_r rides along in shared memory (q_g).
  struct Item {
    int b0;  // < 2^31 half-blocks per tensor (validate_io)
    int nblk;
    uint32_t row;
  };
  auto item_of = [&](const QTensor& T, int li) -> Item {
    Item x;
    if (RI == 2 && T.hpr) {
      x.row = (uint32_t)(li / T.cpr);
      const int c = li - (int)x.row * T.cpr;
      x.b0 = (int)x.row * T.hpr + c * kTaskBlocks;
      x.nblk = min(kTaskBlocks, T.hpr - c * kTaskBlocks);
    } else {
      x.row = 0;
      x.b0 = li * kTaskBlocks;
      x.nblk = (int)min((int64_t)kTaskBlocks, T.nb - x.b0);
    }
    return x;
  };
  // Stage s of this warp holds one item.  Lane l copies its own blocks
  // l, l+32, ... (2 x 16-B LDGSTS each) and later reads back only what it
  // copied, so no cross-lane sync is needed; one commit group per stage
  // (empty groups past the end keep the group count uniform).
  auto issue = [&](int li, int ti, int s) {
    const QTensor& T = p.t[ti];
    const Item x = item_of(T, li);
    const uint8_t* src = T.in + (int64_t)x.b0 * 32;
#pragma unroll
    for (int u = 0; u < kBPL; u++) {
      const int j = u * 32 + lane;
      if (j < x.nblk) {
        cp_async16(&buf[w][s][2 * j], src + j * 32);
        cp_async16(&buf[w][s][2 * j + 1], src + j * 32 + 16);
      }
    }
  };
  auto gscale = [&](int ti, bool report) -> float {
    if (p.gmode == 3) {  // peer-memory exchange (§5b): wait for every rank, then the max
      for (uint32_t spins = 0;; spins++) {
        // >= (mod 2^32): a rank may already have published the NEXT step's
        // flag (it needs nothing from this launch to get there); its slots for
        // this step stay intact in the other parity
        const bool ok = lane >= p.xw || (int32_t)(ld_acquire_sys(p.xin_flag + lane) - p.xepoch_in) >= 0;
        if (__all_sync(0xFFFFFFFFu, ok)) break;
        if (spins == (1u << 25)) {  // ~10 s: a rank never published (watchdog, not a hang)
          if (lane == 0) atomicOr(p.flags, kFlagExchangeTimeout);
          break;
        }
        __nanosleep(256);
      }
      const uint32_t v = lane < p.xw ? ld_relaxed_sys(p.xin + p.t[ti].xslot * kMaxPeers + lane) : 0u;
      return global_scale(__reduce_max_sync(0xFFFFFFFFu, v), p.flags, report, p.g_numer);
    }
    if (p.gmode != 1) return 1.0f;  // 0: G = 1; 2: per-row G, read per block
    return global_scale(__ldg(p.t[ti].amax), p.flags, report, p.g_numer);
  };
  // Dynamic scheduling: counter c hands out units c, c + kCounters, ... ; warp
  // gw draws from counter gw % kCounters, so warps the arbiter favours simply
  // take more units and every warp finishes at about the same time.  Lane 0
  // draws each ticket one unit ahead (`pend`), so the atomic's latency hides
  // under the current unit.  A plain unit is p.ipu items; a row-fused unit is
  // `cpu` consecutive chunks of one row, whose global scale the warp first
  // computes from the whole row (one coalesced pass; the chunks' own reads
  // then hit L2).  Each warp's units increase, so the tensor lookup only
  // moves forward.  Unit and item indices are 32-bit (the host splits
  // batches before 2^31).
  const int cidx = gw % kCounters;
  bool exhausted = false;
  const int nunits = (int)p.ntasks;
  int tj = 0;
  int un_li = 0, un_end = 0, un_pt = 0;  // current plain unit: items [un_li, un_end), its partial
  uint32_t pend = 0;
  if (lane == 0) pend = atomicAdd(p.ctr + cidx, 1u);
  // RI == 2 kernels: the current row-fused unit (chunks [c, ce) of row `row`, scale
  // g still to hand out) lives in shared memory, off the register budget
  struct RowUnit {
    int c, ce;
    uint32_t row;
    float g;
  };
  __shared__ RowUnit ru[RI == 2 ? kWarps : 1];
  __shared__ float q_g[RI == 2 ? kWarps : 1][kStages];
  if (RI == 2) {
    if (lane == 0) ru[w] = RowUnit{0, 0, 0u, 1.0f};
    __syncwarp();
  }
  // next item: its local index (-1 when exhausted), tensor (gti) and the
  // partial to flush after it (gpt, -1 if the unit continues)
  auto grab = [&](int s, int& gti, int& gpt) -> int {
    if constexpr (RI == 2) {
      __syncwarp();
      const RowUnit cur = ru[w];
      if (cur.c < cur.ce) {  // next chunk of the current row
        const QTensor& T = p.t[tj];
        __syncwarp();
        if (lane == 0) {
          ru[w].c = cur.c + 1;
          q_g[w][s] = cur.g;
        }
        const int li = (int)cur.row * T.cpr + cur.c;
        gti = tj;
        gpt = T.part0 + li;
        return li;
      }
    }
    if (un_li < un_end) {  // next item of the current plain unit
      gti = tj;
      const int li = un_li++;
      gpt = un_li == un_end ? un_pt : -1;
      return li;
    }
    if (exhausted) return -1;
    const uint32_t idx = __shfl_sync(0xFFFFFFFFu, pend, 0);
    const int64_t u = cidx + (int64_t)idx * kCounters;
    if (u >= nunits) {
      exhausted = true;
      return -1;
    }
    if (lane == 0) pend = atomicAdd(p.ctr + cidx, 1u);  // the ticket after this one
    tj = locate_task(p, u, tj);
    const QTensor& T = p.t[tj];
    const int k = (int)(u - T.task0);
    gti = tj;
    if constexpr (RI == 2) {
      if (T.hpr) {  // row-fused unit: row k / upr, chunk group k % upr
        const uint32_t row = (uint32_t)(k / T.upr);
        const int c = (k - (int)row * T.upr) * T.cpu;
        const float g = row_global_scale(T, row, lane, p.flags, p.g_numer);
        if (lane == 0 && c == 0) T.g_out[row] = g;
        __syncwarp();
        if (lane == 0) {
          ru[w] = RowUnit{c + 1, min(c + T.cpu, T.cpr), row, g};
          q_g[w][s] = g;
        }
        const int li = (int)row * T.cpr + c;
        gpt = T.part0 + li;
        return li;
      }
    }
    const int items = (int)((T.nb + kTaskBlocks - 1) / kTaskBlocks);
    const int li = k * p.ipu;
    un_end = min(li + p.ipu, items);
    un_li = li + 1;
    un_pt = T.part0 + k;
    gpt = un_li == un_end ? un_pt : -1;
    return li;
  };

  // prologue: kStages items in flight
  int q_li[kStages], q_ti[kStages], q_pt[kStages];
#pragma unroll
  for (int k = 0; k < kStages; k++) {
    int gti = tj, gpt = -1;
    const int li = grab(k, gti, gpt);
    if (li >= 0) issue(li, gti, k);
    q_li[k] = li;
    q_ti[k] = gti;
    q_pt[k] = gpt;
    cp_async_commit();
  }
  int s = 0;
#ifdef SS_COUNT_EVALS
  unsigned long long n_evals = 0;  // per warp (all lanes count the same)
#endif
  // global scale of the current item's tensor, recomputed when the tensor changes
  int cur_ti = -1;
  float G = 1.0f;
  double sb = 0.0, sc = 0.0;  // this lane's error sums over the current unit
  int tt = 0;                 // trailing amax: the fold's task cursor (warp-uniform, moves forward)
  while (q_li[0] >= 0) {
    const int li = q_li[0];
    const int ti = q_ti[0];
    const int pt = q_pt[0];
    const QTensor& T = p.t[ti];
    const Item x = item_of(T, li);
    const int b0 = x.b0;  // first half-block of the item
    const int nblk = x.nblk;
    if (RI == 2 && T.hpr) {  // row-fused: this item's G_r (the next plain item reloads G)
      __syncwarp();
      G = q_g[w][s];
      cur_ti = -1;
    } else if (ti != cur_ti) {  // warp-uniform; a tensor's item 0 always lands here
      cur_ti = ti;
      if constexpr (AF) {  // wait until every amax unit of the tensor has been folded in
#ifdef SS_AF_TRACE
        const unsigned long long t0 = gtime();
#endif
        // watchdog: the amax warps never wait, so this only trips on a stalled GPU
        for (uint32_t spins = 0; ld_acquire_gpu(p.done + ti) < (uint32_t)T.na; spins++) {
          if (spins == (1u << 25)) {  // ~10 s of 256-ns sleeps
            if (lane == 0) atomicOr(p.flags, kFlagAmaxTimeout);
            break;
          }
          __nanosleep(256);
        }
#ifdef SS_AF_TRACE
        if (lane == 0) atomicAdd(p.evals + 2, gtime() - t0);
#endif
        G = p.gmode == 3 ? gscale(ti, li == 0 && lane == 0)  // exchange: the ranks' amaxes
                         : global_scale(ld_relaxed_gpu(T.amax), p.flags, li == 0 && lane == 0, p.g_numer);
      } else {
        G = gscale(ti, li == 0 && lane == 0);
      }
      if (li == 0 && lane == 0 && T.g_out && p.gmode != 2) *T.g_out = G;
    }

    cp_async_wait<kStages - 1>();  // this lane's copies of stage s have landed
    int8_t* offsets = T.offsets ? T.offsets + b0 / kHalves : nullptr;
    float2* err = T.err ? T.err + b0 / kHalves : nullptr;
    // the item's output streams, so a block's stores index them with 32-bit j
    uint2* codes_it = T.codes + b0;
    uint8_t* scales_it = T.scales + b0 / kHalves;
    const uint64_t GG = pack2(G, G);

    // both blocks of a lane in one unrolled body for the windows where that
    // measured faster (r = 2: -2 %, [-2, 6]: -1.4 %; r = 1 and r >= 3 slower,
    // profiles/r02/ab4_unroll.md)
    constexpr int kUnrollU = (NEG == 2 && (POS == 2 || POS == 6)) ? kBPL : 1;
#pragma unroll kUnrollU
    for (int u = 0; u < kBPL; u++) {
      const int j = u * 32 + lane;          // half-block within the item
      const bool active = j < nblk;
      const bool writer = (lane & (kHalves - 1)) == 0;  // owns the scale block
      // scale-block index within the tensor; its row (per-row G, swizzled layout)
      const uint32_t sbk = RI ? (uint32_t)(b0 + min(j, nblk - 1)) / kHalves : (uint32_t)(b0 + j) / kHalves;
      uint32_t row = x.row;
      uint64_t Gb = GG;
      if (RI && !(RI == 2 && T.hpr) && (T.g_row || T.swz)) {  // warp-uniform
        row = div_rows(sbk, T.nbr, T.nbr_magic);
        if (T.g_row) {
          const float gr = __ldg(T.g_row + row);
          Gb = pack2(gr, gr);
        }
      }
      // a1 + a3: bf16 -> f32 is exact; y = RN(x * G)
      const uint4 v0 = buf[w][s][2 * j], v1 = buf[w][s][2 * j + 1];
      const uint32_t wd[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
      float y[16];
      uint64_t y2[8];
#pragma unroll
      for (int k = 0; k < 8; k++) {
        y2[k] = fmul2(bf16x2_to_f32x2(wd[k]), Gb);
        unpack2(y2[k], y[2 * k], y[2 * k + 1]);
      }
      // a4: block max-abs scale code c0 (Alg. 1 lines 1-2)
      float m = 0.0f;
#pragma unroll
      for (int i = 0; i < 16; i++) m = fmaxf(m, fabsf(y[i]));
#pragma unroll
      for (int o = 1; o < kHalves; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
      const float v = __fmul_rn(m, kinv);
      const int c0 = F::SF ? (int)ue8m0_code(v) : (int)e4m3_code(v);
      const uint4* base = F::SF ? tab + Pad + c0 : tab + (c0 ? TabW : 0) + Pad + c0;

      // a5 + a6: candidate search (Alg. 1 lines 5-10).  bidx = the winner's
      // offset into base (its table entry gives code and rho at emit time).
      float best, loss0;
      int bidx;
      if constexpr (NEG >= 0) {
        // f = 0, 1, ..., POS, then -1, ..., -(kPruneFrom - 1): the
        // unconditional candidates, in chunks of CI whose loss loops are
        // interleaved (the selection updates applied in scan order: "<" on
        // the positive side, "<=" on the negative side, R4); then the pruned
        // negative side
        constexpr int NN = NEG < kPruneFrom - 1 ? NEG : kPruneFrom - 1;
        constexpr int NC = 1 + POS + NN;
        constexpr int CI = SS_CILP < NC ? SS_CILP : NC;
        auto off = [](int i) { return i <= POS ? i : POS - i; };  // candidate i -> offset f
#pragma unroll
        for (int i0 = 0; i0 < NC; i0 += CI) {
          uint4 e[CI];
          float l[CI];
#pragma unroll
          for (int c = 0; c < CI; c++) e[c] = base[off(i0 + c < NC ? i0 + c : NC - 1)];
          if constexpr (FMT == kFmtNVFP4) {
            cand_loss_n<CI>(y2, y, e, l);
#ifdef SS_CORE_REPEAT  // tools only: evaluate the unconditional candidates twice (marginal cost per pair)
            {
              uint4 e2[CI];
              float l2[CI];
              uint32_t one;
              asm volatile("mov.b32 %0, 0x3f800000;" : "=r"(one));
#pragma unroll
              for (int c = 0; c < CI; c++) {
                e2[c] = e[c];
                e2[c].x = __float_as_uint(__fmul_rn(__uint_as_float(e[c].x), __uint_as_float(one)));
                e2[c].y = e2[c].x;
              }
              cand_loss_n<CI>(y2, y, e2, l2);
#pragma unroll
              for (int c = 0; c < CI; c++) l[c] = fminf(l[c], l2[c]);
            }
#endif
          } else {
#pragma unroll
            for (int c = 0; c < CI; c++) l[c] = block_loss<FMT>(y2, y, e[c]);
          }
          SS_COUNT(NC - i0 < CI ? NC - i0 : CI);
#pragma unroll
          for (int c = 0; c < CI; c++) {
            const int i = i0 + c;
            if (i >= NC) break;
            if (i == 0) {
              best = l[c];
              loss0 = l[c];  // err_base: the max-abs scale (f = 0)
              bidx = 0;
            } else {
              const bool t_ = i <= POS ? l[c] < best : l[c] <= best;
              best = t_ ? l[c] : best;
              bidx = t_ ? off(i) : bidx;
            }
          }
        }
#pragma unroll
        for (int f = NN + 1; f <= NEG; f++) SS_TAKE_NEG(-f)
      } else {
        best = block_loss<FMT>(y2, y, base[0]);
        SS_COUNT(1);
        loss0 = best;  // err_base: the max-abs scale (f = 0)
        bidx = 0;
        // runtime window; skip offsets that are clamped duplicates for every lane
        const int lo = __reduce_min_sync(0xFFFFFFFFu, F::SF ? -c0 : (c0 ? 1 : 0) - c0);
        const int hi = __reduce_max_sync(0xFFFFFFFFu, F::kMaxCode - c0);
        const int fneg = max(p.fmin, lo), fpos = min(p.fmax, hi);
#pragma unroll 1
        for (int f = 1; f <= fpos; f++) SS_TAKE(f, <)
#pragma unroll 1
        for (int f = -1; f >= fneg; f--) {
          if (f > -kPruneFrom) {
            SS_TAKE(f, <=)
          } else {
            SS_TAKE_NEG(f)
          }
        }
      }

      // a7: emit the winner: codes of t = y * rho*, scale byte, offset, errors
      const uint4 eb = base[bidx];
      const uint32_t code = eb.z >> 16;
      const uint64_t rr = pack2u(eb.x, eb.x);
      float t[16];
#pragma unroll
      for (int k = 0; k < 8; k++) unpack2(fmul2(y2[k], rr), t[2 * k], t[2 * k + 1]);
      if (active) {
        const int64_t hb = b0 + j;  // half-block index within the tensor
        if constexpr (F::VF == 0) {
          uint2 cw;
          cw.x = e2m1_pack8(t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7]);
          cw.y = e2m1_pack8(t[8], t[9], t[10], t[11], t[12], t[13], t[14], t[15]);
          __stcs(codes_it + j, cw);
        } else {  // E2M3: one code per byte
          uint32_t cw[4];
#pragma unroll
          for (int k = 0; k < 4; k++)
            cw[k] = e2m3_pack2(t[4 * k], t[4 * k + 1]) | (e2m3_pack2(t[4 * k + 2], t[4 * k + 3]) << 16);
          __stcs(reinterpret_cast<uint4*>(T.codes) + hb, make_uint4(cw[0], cw[1], cw[2], cw[3]));
        }
        if (writer) {
          if (!RI || !T.swz) {
            scales_it[j / kHalves] = (uint8_t)code;
          } else {
            T.scales[swizzled_scale_offset(row, sbk - row * T.nbr, T.nkt)] = (uint8_t)code;
          }
          const int jb = j / kHalves;  // scale block within the item
          if (offsets) offsets[jb] = (int8_t)((int)code - c0);
          if (err) __stcs(err + jb, make_float2(best, loss0));
          sb += (double)best;
          sc += (double)loss0;
        }
      }
    }
    {  // refill stage s with the next item drawn (always commit: uniform group count)
      int gti = tj, gpt = -1;
      const int nl = grab(s, gti, gpt);
      if (nl >= 0) issue(nl, gti, s);
      cp_async_commit();
#pragma unroll
      for (int k = 0; k + 1 < kStages; k++) {
        q_li[k] = q_li[k + 1];
        q_ti[k] = q_ti[k + 1];
        q_pt[k] = q_pt[k + 1];
      }
      q_li[kStages - 1] = nl;
      q_ti[kStages - 1] = gti;
      q_pt[kStages - 1] = gpt;
    }
    if (pt >= 0) {  // the unit's last item: its partial (fixed lane tree); reduced by sums_kernel
      // trailing amax (§4.2c): the unit's share of the next batch's amax
      if (AF && p.ntrail) trail_fold(p, T.task0 + (pt - T.part0), tt, lane);
      if (T.sums) {
        sb = warp_sum(sb);
        sc = warp_sum(sc);
        if (lane == 0) p.part1[pt] = make_double2(sb, sc);
      }
      sb = 0.0;
      sc = 0.0;
    }

    s = s + 1 == kStages ? 0 : s + 1;
  }
#ifdef SS_AF_TRACE
  if (AF && lane == 0) atomicMax(p.evals + 3, gtime());
#endif
#ifdef SS_COUNT_EVALS
  if (lane == 0 && p.evals) atomicAdd(p.evals, n_evals * 32ull / (unsigned long long)kHalves);
#endif
  // the last warp of the grid to finish re-arms the counters for the next launch
  if (lane == 0) {
    __threadfence();
    if (atomicAdd(p.ctr + kCounters, 1u) == gridDim.x * kWarps - 1) {
      for (int c = 0; c < kCounters; c++) p.ctr[c] = 0u;
      if (AF) {
        for (int i = 0; i < p.n; i++) p.done[i] = 0u;
        p.done[kMaxTensors] = 0u;
        p.done[kMaxTensors + 1] = 0u;
      }
      p.ctr[kCounters] = 0u;
    }
  }
}

}  // namespace ss
