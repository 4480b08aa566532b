// odpo_psync.cuh -- the pair-synchronous split-V schedule (ODPO_SCHED_PSYNC) of the scaled
// Online-DPO loss call (VERDICT r1 "next" item 3).
//
// The scaled gradient dlogits = coef_b (softmax - onehot) needs the pair's coefficient, i.e.
// BOTH sequences' log-probs, before any row of the pair can be written.  FUSED dispatches rows
// adaptively and re-reads a pair's rows from HBM (2R+1W) because the pair completes too long
// after its rows were read.  Here the WHOLE grid works on one pair at a time: the pair's 2T rows,
// flattened into one vector range, are cut into G equal contiguous pieces, CTA j always taking
// piece j.  So the pair's forward pass completes within about one piece-time of its start, and
// CTA j runs
//
//      F(0) F(1) .. F(D-1)  F(D) B(0)  F(D+1) B(1)  ...  B(P-1)
//
// (F = forward of its piece of a pair, B = backward, D = the lag in pairs): the backward of pair
// p trails its forward by D pairs, (D + 1) pairs of logits are live, and they fit in L2 for
// TLDR-like shapes, so the backward re-read is an L2 hit and the HBM traffic is 1R+1W.
//
// Per piece: at most two row segments.  A forward piece leaves one (m, r, x_tok, owns) partial
// per segment in a global window; the CTA that completes the pair (arrival counter) merges each
// row's partials in piece order (= vocabulary order: deterministic), writes the row statistics
// and runs pair_reduce_warp (S3/S4), which publishes the coefficients and pair_ready.  A backward
// piece waits for pair_ready (acquire), reads its rows' constants and writes its dlogits.  Every
// CTA waits only on pairs whose forward pieces it has itself finished and whose other pieces
// never wait, so the schedule needs all CTAs co-resident: it is launched cooperatively.
#pragma once

namespace odpo {

constexpr int kPsNW = 8;                    // consumer warps
constexpr int kPsNT = kPsNW * 32;           // consumer threads
constexpr int kPsStages = 4;                // TMA ring stages of kChunk bytes
constexpr int kPsThreads = kPsNT + 32;      // + the producer warp
constexpr int kPsWin = kPsWinPairs;         // pairs in the partial window (odpo.cu: workspace)
constexpr int kPsMaxG = kPsMaxGrid;         // max grid (window sizing)
constexpr int kPsSmem = kPsStages * kChunk;
constexpr int kPsUB = kCV / kPsNT;          // 16-byte vectors per consumer thread per chunk
static_assert(kCV % kPsNT == 0, "chunk must split evenly over the consumers");

// piece j of a pair: flattened vectors [ps_lo(j), ps_lo(j + 1)) of 2T * nvec
__device__ __forceinline__ int64_t ps_lo(int64_t N, int64_t G, int64_t j) { return N * j / G; }

// row r (0 <= r < 2T) of pair p -> (sequence, t); r < T: the chosen sequence
__device__ __forceinline__ void ps_row(const LossArgs& a, int64_t p, int64_t r, int64_t& s,
                                       int64_t& t) {
  int64_t c, rj;
  pair_seqs(a, p, c, rj);
  s = r < a.T ? c : rj;
  t = r < a.T ? r : r - a.T;
}

// Stage metadata (written by the producer before the stage's full barrier).
struct PsStage {
  int32_t kind;     // K_F / K_B / K_END
  int32_t seg;      // segment (0 or 1) of the piece
  int32_t last;     // last chunk of the segment
  int32_t lastseg;  // the piece's last segment
  int32_t v0, nv;   // vector range of this chunk within its row
  int64_t p, g;     // pair, row id s*T + t (-1: the pair member is out of range)
  int32_t first;    // first chunk of the piece
  int32_t live;     // the row has mask = 1 (else nothing was loaded)
};

template <int DT>
__global__ void __launch_bounds__(kPsThreads, 1) k_psync(LossArgs a, int D) {
  constexpr int N = Traits<DT>::N;
  extern __shared__ __align__(1024) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[kPsStages], empty[kPsStages];
  __shared__ PsStage meta[kPsStages];
  __shared__ float wm[kPsNW], wr[kPsNW];
  __shared__ float s_xt;
  __shared__ int s_own;
  __shared__ int s_reduce;
  __shared__ float bc[2], bcoef[2], bgtok[2], bm[2];   // backward constants per segment
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kPsStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kPsNW);
    }
    mbar_fence_init();
    s_own = 0;
    s_xt = 0.f;
  }
  __syncthreads();
  const uint32_t full_s = smem_u32(full), empty_s = smem_u32(empty), ring_s = smem_u32(ring);
  const int64_t G = gridDim.x, j = blockIdx.x;
  const int nvec = (int)(a.V / N);
  const int64_t Np = 2 * a.T * nvec;          // vectors per pair
  const int64_t lo = ps_lo(Np, G, j), hi = ps_lo(Np, G, j + 1);
  const float k2 = a.invT * kLog2e;
  const int64_t nsteps = a.P + D;

  if (warp == kPsNW) {
    // ================= producer: the piece's chunks, item by item, into the ring
    if (lane == 0) {
      const uint64_t pol_keep = policy_evict_last(), pol_drop = policy_evict_first();
      int st = 0;
      uint32_t ph = 0;
      auto item = [&](int kind, int64_t p) {
        bool first = true;
        int seg = 0;
        for (int64_t v = lo; v < hi; ++seg) {
          const int64_t r = v / nvec;
          const int64_t vend = min(hi, (r + 1) * nvec);
          int64_t s, t;
          ps_row(a, p, r, s, t);
          const bool live = s >= 0 && a.mask[s * a.T + t] != 0;
          const char* row = row_ptr(a, s < 0 ? 0 : s, t);
          for (int64_t c = v; c < vend; c += kCV) {
            const int nv = (int)min((int64_t)kCV, vend - c);
            mbar_wait(empty_s + 8 * st, ph ^ 1u);
            PsStage& M = meta[st];
            M.kind = kind; M.seg = seg; M.p = p; M.g = s < 0 ? -1 : s * a.T + t;
            M.v0 = (int)(c - r * nvec); M.nv = nv; M.live = live;
            M.last = c + kCV >= vend; M.lastseg = vend >= hi; M.first = first;
            first = false;
            if (live) {
              mbar_arrive_tx(full_s + 8 * st, (uint32_t)nv * 16u);
              tma_load_1d(ring_s + st * kChunk, row + (size_t)(c - r * nvec) * 16, (uint32_t)nv * 16u,
                          full_s + 8 * st, kind == K_F ? pol_keep : pol_drop);
            } else {
              mbar_arrive(full_s + 8 * st);
            }
            if (++st == kPsStages) { st = 0; ph ^= 1u; }
          }
          v = vend;
        }
      };
      for (int64_t k = 0; k < nsteps; ++k) {
        if (k < a.P) item(K_F, k);
        if (k >= D) item(K_B, k - D);
      }
      mbar_wait(empty_s + 8 * st, ph ^ 1u);
      meta[st].kind = K_END;
      mbar_arrive(full_s + 8 * st);
    }
    return;
  }

  // ================= consumers
  const uint32_t NI = Traits<DT>::kNegInfWord;
  int st = 0;
  uint32_t ph = 0;
  MR s{-INFINITY, 0.f};
  float b_c = 0.f, b_coef = 0.f, b_gtok = 0.f, b_m = 0.f;
  auto cbar = [&]() { asm volatile("bar.sync 1, %0;" ::"n"(kPsNT) : "memory"); };
  for (;;) {
    mbar_wait(full_s + 8 * st, ph);
    const PsStage M = meta[st];
    if (M.kind == K_END) break;
    const uint4* sv = reinterpret_cast<const uint4*>(ring + (size_t)st * kChunk);
    int64_t tok = -1;
    if (M.g >= 0) tok = a.tokens[M.g];
    const int tvec = (tok >= 0 && tok < (int64_t)nvec * N) ? (int)(tok / N) - M.v0 : -1;
    const bool own_tok = M.live && tvec >= 0 && tvec < M.nv && (tvec % kPsNT) == tid;
    if (M.kind == K_F) {
      if (M.live) {
        uint4 v[kPsUB];
#pragma unroll
        for (int u = 0; u < kPsUB; ++u) {
          const int i = tid + u * kPsNT;
          v[u] = i < M.nv ? sv[i] : make_uint4(NI, NI, NI, NI);
        }
        if (tid < M.nv) mr_batch<DT, kPsUB, 0>(v, k2, s.m, s.r);
        if (own_tok) {
          float f[N];
          Traits<DT>::unpack(sv[tvec], f);
          float x = f[0];
#pragma unroll
          for (int q = 1; q < N; ++q) x = (tok % N == q) ? f[q] : x;
          s_xt = x;
          s_own = 1;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty_s + 8 * st);
      if (M.last) {
        // segment done: fixed-order warp then CTA merge -> the segment's partial
        const MR wv = warp_merge(s, k2);
        if (lane == 0) { wm[warp] = wv.m; wr[warp] = wv.r; }
        s = MR{-INFINITY, 0.f};
        cbar();
        if (tid == 0) {
          MR u{-INFINITY, 0.f};
          for (int w = 0; w < kPsNW; ++w) u = mr_merge(u, MR{wm[w], wr[w]}, k2);
          const int own = s_own;
          a.w.psparts[((M.p % kPsWin) * G + j) * 2 + M.seg] =
              make_float4(u.m, u.r, own ? s_xt : 0.f, own ? 1.f : 0.f);
          s_own = 0;
          s_xt = 0.f;
          s_reduce = 0;
          if (M.lastseg) {
            // this piece of pair p is done: count it; the last piece's CTA reduces the pair
            __threadfence();
            const unsigned n = atom_add_acq_rel(&a.w.pair_cnt[M.p], 1u);
            s_reduce = n == (unsigned)(G - 1);
            if (s_reduce) fence_acq_rel_gpu();
          }
        }
        cbar();
        if (M.lastseg && s_reduce) {
          // ---- the pair's reduction: every row merges its pieces' partials in piece order
          const int64_t R2 = 2 * a.T;
          uint32_t fl = 0;
          for (int64_t r = tid; r < R2; r += kPsNT) {
            int64_t sq, t;
            ps_row(a, M.p, r, sq, t);
            if (sq < 0) continue;
            const int64_t g = sq * a.T + t;
            if (!a.mask[g]) continue;
            // pieces covering row r: j0 = the piece holding its first vector, through j1
            const int64_t v0 = r * nvec, v1 = (r + 1) * nvec - 1;
            int64_t j0 = v0 * G / Np, j1 = v1 * G / Np;
            while (ps_lo(Np, G, j0) > v0) --j0;
            while (ps_lo(Np, G, j0 + 1) <= v0) ++j0;
            while (ps_lo(Np, G, j1) > v1) --j1;
            while (ps_lo(Np, G, j1 + 1) <= v1) ++j1;
            MR u{-INFINITY, 0.f};
            float xt = 0.f;
            int owners = 0;
            for (int64_t q = j0; q <= j1; ++q) {
              // the segment of piece q on row r: segment 0 unless piece q starts on an earlier row
              const int sg = (ps_lo(Np, G, q) / nvec == r) ? 0 : 1;
              const float4 pq = __ldcg(&a.w.psparts[((M.p % kPsWin) * G + q) * 2 + sg]);
              u = mr_merge(u, MR{pq.x, pq.y}, k2);
              if (pq.w != 0.f) { xt = pq.z; ++owners; }
            }
            const float l1p = log1pf(u.r);
            float logp = 0.f;
            const int32_t tk = a.tokens[g];
            if (tk < 0 || (int64_t)tk >= a.V || owners != 1) {
              fl |= ODPO_FLAG_TOKEN_RANGE;
            } else {
              logp = __fsub_rn(__fmul_rn(__fsub_rn(xt, u.m), a.invT), l1p);
              if (!isfinite(logp)) fl |= ODPO_FLAG_NONFINITE_LOGIT;
            }
            if (!isfinite(u.m) || !isfinite(u.r)) fl |= ODPO_FLAG_NONFINITE_LOGIT;
            a.w.row_m[g] = u.m;
            a.w.row_l1p[g] = l1p;
            a.w.row_logp[g] = logp;
          }
          flag(a.status, fl);
          __threadfence();
          cbar();
          if (warp == 0) pair_reduce_warp(a, M.p);   // coefficients, stats, pair_ready (release)
          cbar();
        }
      }
    } else {  // K_B
      if (M.first) {
        // wait for the pair's coefficient, then this piece's row constants (<= 2 segments)
        if (tid == 0) {
          while (ld_relaxed(&a.w.pair_ready[M.p]) == 0u) __nanosleep(64);
          fence_acq_rel_gpu();
        }
        cbar();
        if (tid < 2) {
          // segment tid of this piece of pair M.p
          const int64_t v = tid == 0 ? lo : ((lo / nvec) + 1) * nvec;
          if (v < hi) {
            int64_t sq, t;
            ps_row(a, M.p, v / nvec, sq, t);
            float c = INFINITY, cf = 0.f, gt = 0.f, m = 0.f;
            if (sq >= 0) {
              const int64_t g = sq * a.T + t;
              cf = __ldcg(a.w.seq_coef + sq);
              m = __ldcg(a.w.row_m + g);
              const float l1p = __ldcg(a.w.row_l1p + g);
              gt = cf * expm1f(__ldcg(a.w.row_logp + g));
              if (cf != 0.f) c = bwd_const<DT>(m, l1p, k2, cf);
            }
            bc[tid] = c; bcoef[tid] = cf; bgtok[tid] = gt; bm[tid] = m;
          }
        }
        cbar();
      }
      b_c = bc[M.seg]; b_coef = bcoef[M.seg]; b_gtok = bgtok[M.seg]; b_m = bm[M.seg];
      if (M.g >= 0) {
        uint4* vout = reinterpret_cast<uint4*>(drow_ptr(a, M.g / a.T, M.g % a.T)) + M.v0;
#pragma unroll
        for (int u = 0; u < kPsUB; ++u) {
          const int i = tid + u * kPsNT;
          if (i < M.nv) {
            if (!M.live) st16_stream(vout + i, make_uint4(0, 0, 0, 0));   // masked row: zeros
            else st16_stream(vout + i, b_coef < 0.f ? bwd_vec<DT, 0, true>(sv[i], k2, b_c, b_m)
                                                    : bwd_vec<DT, 0, false>(sv[i], k2, b_c, b_m));
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty_s + 8 * st);
      if (own_tok) Traits<DT>::store1(drow_ptr(a, M.g / a.T, M.g % a.T), tok, b_gtok);
    }
    if (++st == kPsStages) { st = 0; ph ^= 1u; }
  }
}

// Rows of sequences that no pair references: zeros (PSYNC streams pairs only).
template <int DT>
__global__ void __launch_bounds__(256) k_zero_unref(LossArgs a) {
  constexpr int N = Traits<DT>::N;
  const int64_t nrows = (int64_t)__ldcg(&a.w.counters[C_NUNREF]) * a.T;
  const int nvec = (int)(a.V / N);
  for (int64_t u = blockIdx.x; u < nrows; u += gridDim.x) {
    const int64_t s = a.w.unref[u / a.T], t = u % a.T;
    uint4* o = reinterpret_cast<uint4*>(drow_ptr(a, s, t));
    for (int i = threadIdx.x; i < nvec; i += blockDim.x) st16_stream(o + i, make_uint4(0, 0, 0, 0));
  }
}

}  // namespace odpo
