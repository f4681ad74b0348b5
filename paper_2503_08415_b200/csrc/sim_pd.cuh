// sim_pd.cuh -- a.9: the disaggregated 1P:1D pair (readings A35, R-PD1..7).
// Included by sim.cu after the shared helpers; one warp simulates one (prefill profile, decode
// profile) point.
//
// P runs prefill-only iterations and emits the first token; at the end-of-prefill
// breakpoint the request joins D's pending FIFO still holding its P blocks.  D pulls
// pending requests FCFS at its boundaries, allocates ceil(p/bs) blocks and starts a p*kvb-byte
// transfer on the FIFO P->D link; the request runs on D from the first D boundary
// >= transfer end; P frees its blocks at its first boundary >= transfer end.  The worker with the
// earlier next boundary is advanced, D first on ties (A2); an idle worker wakes at the earliest
// event that can change its decision.
//
// Data: D's requests live in the warp's slot array, id-sorted: running and preempted requests
// interleave (state per slot), in-flight transfers form the tail.  P's block lists move from a
// per-iteration batch table into a per-warp global ring (segments freed in FIFO = transfer
// order); the pending/transfer FIFO is a per-warp global array of 32-byte entries.
#pragma once
// (included inside namespace ts)

struct FifoEnt {
  u32 id, seg, len, pad;
  i64 join, xend;
};

enum : u32 { ST_RUN = 0, ST_QUEUED = 1, ST_XFER = 2, ST_RUN_RECOMP = 4 };

struct TraceAcc {  // lane-uniform BINNED/FULL trace state of one worker
  u64 tn, bin, acc_bns;
  i64 bin_end;
  u32 acc_max, acc_nit;
};  // (FULL traces keep their FullEnc apart: this struct is copied with a worker's scalars)

__device__ __forceinline__ void trace_flush_bin(TraceAcc &A, tokensim_mem_sample *trc, u64 cap, i64 W, u32 &flags) {
  if (A.tn < cap) {
    if (lane_id() == 0) {
      tokensim_mem_sample s;
      s.t_ns = (i64)A.bin * W;
      s.dur_ns = W;
      s.block_ns = A.acc_bns;
      s.blocks_max = A.acc_max;
      s.n_iter = A.acc_nit;
      trc[A.tn] = s;
    }
  } else {
    flags |= TOKENSIM_PT_TRACE_OVERFLOW;
  }
  ++A.tn;
  ++A.bin;
  A.bin_end += W;
  A.acc_bns = 0;
  A.acc_max = 0;
  A.acc_nit = 0;
}

__device__ __forceinline__ void trace_iter(TraceAcc &A, FullEnc &fe, bool binned, bool full, tokensim_mem_sample *trc,
                                           u64 cap, i64 W, i64 ts, i64 te, u64 blocks, u32 &flags) {
  if (binned) {
    while (A.bin_end <= ts) trace_flush_bin(A, trc, cap, W, flags);
    ++A.acc_nit;
    i64 s = ts;
    while (te > A.bin_end) {
      if (A.bin_end > s) {
        A.acc_bns += blocks * (u64)(A.bin_end - s);
        A.acc_max = max(A.acc_max, (u32)blocks);
      }
      s = A.bin_end;
      trace_flush_bin(A, trc, cap, W, flags);
    }
    if (te > s) {
      A.acc_bns += blocks * (u64)(te - s);
      A.acc_max = max(A.acc_max, (u32)blocks);
    }
  } else if (full) {
    full_trace_put(fe, reinterpret_cast<unsigned char *>(trc), cap * sizeof(tokensim_mem_sample), 1u, ts, te, blocks,
                   flags);
  }
}

// memory trace of a stretch: lanes j < J hold iterations [tsj, tej) with blkj blocks
__device__ __forceinline__ void trace_stretch(TraceAcc &A, FullEnc &fe, bool binned, bool full, tokensim_mem_sample *trc, u64 cap,
                                              i64 W, u32 J, i64 tsj, i64 tej, u64 blkj, u32 &flags) {
  const u32 lane = lane_id();
  const bool lj = lane < J;
  const i64 tend = __shfl_sync(FULLMASK, tej, J - 1), tsl = __shfl_sync(FULLMASK, tsj, J - 1);
  if (binned) {
    while (true) {
      const i64 bstart = A.bin_end - W;
      i64 ov = 0;
      bool cnt_here = false;
      if (lj) {
        const i64 lo = tsj > bstart ? tsj : bstart;
        const i64 hi = tej < A.bin_end ? tej : A.bin_end;
        ov = hi - lo;
        cnt_here = tsj >= bstart && tsj < A.bin_end;
      }
      A.acc_bns += warp_sum64(ov > 0 ? blkj * (u64)ov : 0ull);
      A.acc_max = max(A.acc_max, __reduce_max_sync(FULLMASK, ov > 0 ? (u32)blkj : 0u));
      A.acc_nit += __popc(__ballot_sync(FULLMASK, cnt_here));
      if (tend > A.bin_end || tsl >= A.bin_end) trace_flush_bin(A, trc, cap, W, flags);
      else break;
    }
  } else if (full) {
    full_trace_put(fe, reinterpret_cast<unsigned char *>(trc), cap * sizeof(tokensim_mem_sample), J, tsj, tej, blkj,
                   flags);
  }
}

template <int CAP, bool P2>
__device__ void simulate_pd(const SweepParams &P, u64 j, const WarpSmem &S, unsigned char *pd_smem, u32 *bt) {
  const u32 lane = lane_id();
  const u32 ltm = lanemask_lt();
  const u64 point = P.begin + j * P.stride;
  const Coords cd = decode_point(point, P.n_pol, P.n_rates, P.n_seeds);
  const u32 hwP = cd.hw / P.n_hw, hwD = cd.hw % P.n_hw;
  const DevHP HPP = P.hp[(size_t)hwP * P.n_pol + cd.pol];
  const DevHP HPD = P.hp[(size_t)hwD * P.n_pol + cd.pol];
  const DevPol PL = P.pol[cd.pol];
  const CostK KP = make_costk(P.M, P.MF, P.hw[hwP]);
  const CostK KD = make_costk(P.M, P.MF, P.hw[hwD], P.link_mode, P.preload_buf);
  const u32 g = P.group_of_point_mode ? 0u : cd.rate * P.n_seeds + cd.seed;
  const u32 n = P.n_req;
  const i64 *A = P.arrival + (size_t)g * n;
  const u32 *PR = P.prompt + (size_t)g * n;
  const u32 *OU = P.output + (size_t)g * n;
  tokensim_request_record *rec = P.rec + (size_t)j * n;
  tokensim_mem_sample *trcP = P.trace + (size_t)j * P.trace_nw * P.trace_cap;
  tokensim_mem_sample *trcD = trcP + P.trace_cap;
  tokensim_iter_record *itr = P.itrec + (size_t)j * P.it_cap;
  const BSz B = {PL.bs, PL.bs_sh, PL.bs - 1u, P2 || PL.bs_sh != 0xffffffffu};  // P2: folded to shifts
  const bool SWAPM = PL.preempt == TOKENSIM_SWAP;
  const bool STATICP = PL.kind == TOKENSIM_STATIC;
  const u64 totP = HPP.total_blocks, totD = HPD.total_blocks;
  const u32 nwP = HPP.nwords, nwD = HPD.nwords;
  const u32 btl = P.bt_len;
  const u32 mns = PL.mns, mbt = PL.mbt;
  const i64 wm = (i64)PL.wm;
  const i64 INF = INT64_MAX;
  const long long clk0 = clock64();
  // per-warp extras
  u32 *stt = reinterpret_cast<u32 *>(pd_smem);
  u32 *pid = stt + CAP;
  u32 *pinfo = pid + CAP;
  u32 *ppl = pinfo + CAP;
  u32 *pol = ppl + CAP;
  u32 *bmP = pol + CAP;
  const u32 gwarp = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  u32 *ring = P.pd_ring + (size_t)gwarp * P.pd_ring_len;
  FifoEnt *fifo = reinterpret_cast<FifoEnt *>(P.pd_fifo) + (size_t)gwarp * n;
  const u64 ring_len = P.pd_ring_len;
  u32 *btD = bt;                             // D block tables [CAP][btl]
  u32 *btP = bt + (size_t)CAP * btl;         // P batch block tables [CAP][btl]
  WarpSmem SP = S;                           // P view for the allocator
  SP.id = pid;
  SP.info = pinfo;
  SP.bitmap = bmP;

  // ---- init
  {
    ulonglong2 *r2 = reinterpret_cast<ulonglong2 *>(rec);
    const ulonglong2 z = make_ulonglong2(0ull, 0ull);
    #pragma unroll 1
    for (u32 x = lane; x < 2 * n; x += 32) r2[x] = z;
    #pragma unroll 1
    for (u32 w = lane; w < nwD; w += 32) {
      const u32 fw = (u32)(totD >> 5), tl = (u32)(totD & 31u);
      S.bitmap[w] = w < fw ? 0xffffffffu : (w == fw && tl ? ((1u << tl) - 1u) : 0u);
    }
    #pragma unroll 1
    for (u32 w = lane; w < nwP; w += 32) {
      const u32 fw = (u32)(totP >> 5), tl = (u32)(totP & 31u);
      bmP[w] = w < fw ? 0xffffffffu : (w == fw && tl ? ((1u << tl) - 1u) : 0u);
    }
    #pragma unroll 1
    for (u32 w = lane; w < CAP / 32; w += 32) S.btfree[w] = 0xffffffffu;
    #pragma unroll 1
    for (u32 x = lane; x < CAP; x += 32) pinfo[x] = x;
    __syncwarp();
  }
  i64 tP = 0, tD = 0, link_busy = 0, lastP = 0, lastD = 0, pf_end = INF, xhead_end = INF;
  bool P_idle = false, D_idle = false;
  u64 kP = 0, kD = 0, nfreeP = totP, nfreeD = totD;
  u32 hintP = 0, hintD = 0, arr = 0, adm = 0, n_done = 0;
  u32 nD = 0, nX = 0, nQ = 0, nRun = 0;  // D slots: all / in-flight (tail) / preempted / running
  u32 ftail = 0, fpfree = 0, fdadm = 0, fvis = 0;
  u64 ring_tail = 0;
  Logs L;
  L.ev = P.evlog + (size_t)gwarp * EVCAP;
  L.it = P.itlog + (size_t)gwarp * ITCAP * 4;
  L.itr = itr;
  L.it_cap = P.it_cap;
  L.it_base = 0;
  L.dig_s = 0;
  L.dig_b = 0;
  L.nev = 0;
  L.nit = 0;
  u64 req_iters = 0, npre = 0, swo = 0, swi = 0, nrej_tot = 0, nfin_tot = 0, peakD = 0, bnsD = 0, n_xfer = 0,
      xbytes = 0;
  u32 flags = 0;
  i64 last_fin = 0;
  const bool ff_on = P.ff_enable != 0;
  u32 rminD = 0;              // min rem over D's running slots after the last commit
  u64 ffw = 0, ffk = 0;       // memory-cut retry guard (as in the unified worker)
  u64 ff_iters = 0, ff_runs = 0;
  u64 nit = 0;  // iteration records are kept in processing order across both workers
  u64 cyc_ffD = 0, cyc_failD = 0, cyc_normD = 0;
  const bool BINNED = P.trace_mode == TOKENSIM_TRACE_BINNED;
  const bool FULLT = P.trace_mode == TOKENSIM_TRACE_FULL;
  const i64 W = (i64)P.bin_ns;
  TraceAcc TA[2] = {{0, 0, 0, W, 0, 0}, {0, 0, 0, W, 0, 0}};
  FullEnc FE[2] = {{0, 0, 0, 0, 0, 0}, {0, 0, 0, 0, 0, 0}};
  // request window (P side)
  u32 win = 0;
  i64 wa = INT64_MAX;
  u32 wp = 0, wo = 0;
  auto load_win = [&](u32 base) {
    win = base;
    const u32 i = base + lane;
    wa = i < n ? A[i] : INT64_MAX;
    wp = i < n ? PR[i] : 0u;
    wo = i < n ? OU[i] : 0u;
  };
  load_win(0);
  auto fold_iter = [&](u64 kk, u32 worker, i64 ts, i64 T, u64 Sp, u64 D_, u64 Np, u64 Cd, u64 m, u64 nres,
                       u64 nadm, u64 nrej, u64 nfin, u64 blocks) {
    it_reserve(L, 1);
    if (lane == 0) it_put(L, 0, kk | ((u64)worker << 40), ts, T, Np, Cd, blocks, Sp, D_, m, nres, nadm, nfin, nrej);
    L.nit += 1;
    ++nit;
  };
  auto xfer_ns = [&](u32 p) -> i64 {
    const u64 bytes = (u64)p * P.M.kvb;
    return (i64)floor(__dadd_rn(__dmul_rn(__dmul_rn(__ull2double_rn(bytes), P.pd_link_inv), 1e9), 0.5));
  };

  while (true) {
    if (n_done == n) break;
    const i64 tnext = tP < tD ? tP : tD;
    if (tnext == INF) {
      flags |= TOKENSIM_PT_INTERNAL_ERROR;  // both workers wait: cannot happen under validation
      break;
    }
    if (P.horizon >= 0 && tnext >= P.horizon) {
      flags |= TOKENSIM_PT_HORIZON_HIT;
      break;
    }
    if (tD <= tP) {
      // ============================================================ D boundary
      const i64 t = tD;
      long long cD = prof_clock();  // observability: cycles by path (point profile)
      // 1. finished transfers become runnable (the in-flight tail completes in FIFO order)
      while (nX > 0 && xhead_end <= t) {
        const u32 pos = nD - nX;
        if (lane == 0) stt[pos] = ST_RUN;
        --nX;
        ++nRun;
        xhead_end = nX ? fifo[fdadm - nX].xend : INF;
      }
      __syncwarp();
      // ---------------------------------------------------------- D fast-forward (H3)
      // Quiescent decode stretch on D: nothing completes a transfer, nothing is pulled or
      // resumed, nothing is preempted, and P (which may push pending requests) has no boundary
      // before the stretch's iterations; the last iteration may finish requests.
      if (ff_on && nRun > 0 && rminD >= 2 && (nfreeD > ffw || kD >= ffk)) {
        bool quiet = true, mem_check = false;
        u32 need_h = 0;
        i64 join_cut = INF;
        const u32 nA0 = nD - nX;
        if (nQ > 0) {
          // first preempted slot = the resume head
          u32 qpos = 0;
          #pragma unroll 1
          for (u32 b0 = 0; b0 < nA0; b0 += 32) {
            const u32 jj = b0 + lane;
            const u32 qb = __ballot_sync(FULLMASK, jj < nA0 && stt[jj] == ST_QUEUED);
            if (qb) {
              qpos = b0 + (u32)(__ffs(qb) - 1);
              break;
            }
          }
          u32 tokq;
          if (SWAPM) {
            const u32 c = S.ctx[qpos];
            need_h = B.cdiv(c) + (B.mod(c) == 0 ? 1u : 0u);
            tokq = 1;
          } else {
            const u32 id = S.id[qpos];
            tokq = PR[id] + (OU[id] - S.rem[qpos]);
            need_h = B.cdiv(tokq);
          }
          if (!((u64)nRun + nX + 1 > mns || (u64)nRun + tokq > mbt)) {
            mem_check = true;
            if ((i64)nfreeD - (i64)nRun - (i64)need_h >= wm) quiet = false;  // resume is certain
          }
        } else if (!STATICP) {
          if (fdadm < ftail) {
            const i64 jh = fifo[fdadm].join;
            if (jh <= t) {  // a visible pending head: blocked now => blocked for the stretch
              need_h = B.cdiv(PR[fifo[fdadm].id]);
              if (!((u64)nRun + nX + 1 > mns)) {
                mem_check = true;
                if ((i64)nfreeD - (i64)nRun - (i64)need_h >= wm) quiet = false;
              }
            } else {
              join_cut = jh;  // the head becomes visible later
            }
          }
        }
        if (quiet) {
          S.scratch[lane] = 0;
          S.scratch[32 + lane] = 0;
          __syncwarp();
          u64 cdp0 = 0;
          u32 rmn = 0xffffffffu;
          i64 lmin = INF;
          #pragma unroll 1
          for (u32 b0 = 0; b0 < nA0; b0 += 32) {
            const u32 jj = b0 + lane;
            u32 key = 64u + lane;
            if (jj < nA0 && stt[jj] == ST_RUN) {
              const u32 c = S.ctx[jj];
              cdp0 += c + 1;
              rmn = min(rmn, S.rem[jj]);
              const i64 lt = S.last[jj];
              lmin = lt < lmin ? lt : lmin;
              const u32 r = B.mod(c);
              const u32 j0 = r ? B.bs - r : 0u;
              if (j0 < 32) key = j0;
            }
            const u32 peers = __match_any_sync(FULLMASK, key);
            if (key < 32 && (peers & ltm) == 0u) {
              S.scratch[key] += __popc(peers);
              S.scratch[32 + key] = peers;
            }
            __syncwarp();
          }
          const u64 Cd0 = warp_sum64(cdp0);
          const u32 rm = __reduce_min_sync(FULLMASK, rmn);
          i64 lm = lmin;
#pragma unroll
          for (u32 o = 16; o; o >>= 1) {
            const i64 y = __shfl_xor_sync(FULLMASK, lm, o);
            lm = y < lm ? y : lm;
          }
          const u32 nj = S.scratch[B.bs >= 32 ? lane : B.mod(lane)];
          const u32 Aj = scan_incl(nj);
          const u64 Cdj = Cd0 + (u64)lane * nRun;
          const i64 Tj = iter_time_ns(KD, 0, 0, 0, nRun, Cdj, 0);
          const i64 tej = t + scan_incl_i64(Tj);
          const i64 tsj = tej - Tj;
          bool ok = ((u64)Aj <= nfreeD) && (Aj <= (u32)CAP) && (lane < rm);
          if (lane > 0) {
            if (P.horizon >= 0 && tsj >= P.horizon) ok = false;
            if (tsj >= xhead_end || tsj >= join_cut || tsj > tP) ok = false;
          }
          if (mem_check) {
            const u64 fr = nfreeD - (u64)__shfl_sync(FULLMASK, Aj, 0);
            if (!((i64)fr - (i64)need_h < wm)) ok = false;
          }
          const u32 okm = __ballot_sync(FULLMASK, ok);
          const u32 J = (~okm == 0u) ? 32u : (u32)(__ffs(~okm) - 1);
          const u32 memcut = __ballot_sync(FULLMASK, !((u64)Aj <= nfreeD));
          if (J < 2 && memcut && (u32)(__ffs(memcut) - 1) < 2) {
            ffw = nfreeD;
            ffk = kD + 4;
          }
          if (J >= 2) {
            const u32 Ktot = __shfl_sync(FULLMASK, Aj, J - 1);
            __syncwarp();
            S.scratch[lane] = Aj - nj;  // bucket cursors
            __syncwarp();
            bool done_alloc = Ktot == 0;
            if (!done_alloc && nA0 <= 32 && Ktot <= 32 && hintD < nwD) {
              const u32 wi = hintD + lane;
              u32 word = wi < nwD ? S.bitmap[wi] : 0u;
              const u32 cw = __popc(word);
              const u32 cum = scan_incl(cw);
              if (__shfl_sync(FULLMASK, cum, 31) >= Ktot) {
                ev_reserve(L, 32);
                const bool act = lane < Ktot;
                const u32 o = act ? lane : 0u;
                u32 jb = 0;
#pragma unroll
                for (u32 st = 16; st; st >>= 1) {
                  const u32 v = __shfl_sync(FULLMASK, Aj, jb + st - 1);
                  if (v <= o) jb += st;
                }
                const u32 excl = __shfl_sync(FULLMASK, Aj - nj, jb);
                u32 lo = 0;
#pragma unroll
                for (u32 st = 16; st; st >>= 1) {
                  const u32 v = __shfl_sync(FULLMASK, cum, lo + st - 1);
                  if (v <= o) lo += st;
                }
                const u32 wv = __shfl_sync(FULLMASK, word, lo);
                const u32 bv = __shfl_sync(FULLMASK, cum - cw, lo);
                if (act) {
                  const u32 mask = S.scratch[32 + (B.bs >= 32 ? jb : B.mod(jb))];
                  const u32 pos = select_bit(mask, o - excl);
                  const u32 blk = (hintD + lo) * 32 + select_bit(wv, o - bv);
                  btD[(size_t)(S.info[pos] & 0xffffu) * btl + B.div(S.ctx[pos] + jb)] = blk;
                  ev_put(L, o, kD + jb, 3, S.id[pos], blk);
                }
                L.nev += Ktot;
                const u32 before = cum - cw;
                const u32 tk = Ktot > before ? min(cw, Ktot - before) : 0u;
                if (tk && wi < nwD) {
                  word = clear_lowest(word, tk, cw);
                  S.bitmap[wi] = word;
                }
                const u32 nz = __ballot_sync(FULLMASK, word != 0u);
                hintD = nz ? hintD + (u32)(__ffs(nz) - 1) : hintD + 32;
                __syncwarp();
                done_alloc = true;
              }
            }
            if (!done_alloc) {
              const u32 nrep = B.cdiv(32u);
              #pragma unroll 1
              for (u32 b0 = 0; b0 < nA0; b0 += 32) {
                const u32 jj = b0 + lane;
                const bool run = jj < nA0 && stt[jj] == ST_RUN;
                const u32 c = run ? S.ctx[jj] : 0u;
                const u32 r = B.mod(c);
                u32 jx = r ? B.bs - r : 0u;
                #pragma unroll 1
                for (u32 rep = 0; rep < nrep; ++rep, jx += B.bs) {
                  const bool v = run && jx < J;
                  const u32 key = v ? jx : 64u + lane;
                  const u32 peers = __match_any_sync(FULLMASK, key);
                  u32 base = 0;
                  if (v) base = S.scratch[jx];
                  __syncwarp();
                  if (v) {
                    const u32 e = base + __popc(peers & ltm);
                    S.req_cum[e] = e + 1;
                    S.req_pt[e] = jj | (jx << 10) | (B.div(c + jx) << 15);
                    if ((peers & ltm) == 0u) S.scratch[jx] = base + __popc(peers);
                  }
                  __syncwarp();
                }
              }
              if (!alloc_ordered(S, Ktot, Ktot, btD, btl, kD, 2, L, hintD, nwD)) {
                flags |= TOKENSIM_PT_INTERNAL_ERROR;
                break;
              }
            }
            const u64 blk0 = totD - nfreeD;
            nfreeD -= Ktot;
            const u64 klast = kD + J - 1;
            const i64 tend = __shfl_sync(FULLMASK, tej, J - 1);
            const i64 te0 = __shfl_sync(FULLMASK, tej, 0);
            const bool lj = lane < J;
            i64 tm1 = (lj && lane > 0) ? Tj : 0;  // gaps of iterations 1.. are their T
#pragma unroll
            for (u32 o = 16; o; o >>= 1) {
              const i64 y = __shfl_xor_sync(FULLMASK, tm1, o);
              tm1 = y > tm1 ? y : tm1;
            }
            u32 nfin = 0, first_fin = 0xffffffffu, rmin_l = 0xffffffffu;
            #pragma unroll 1
            for (u32 b0 = 0; b0 < nA0; b0 += 32) {
              const u32 jj = b0 + lane;
              bool fin = false;
              if (jj < nA0 && stt[jj] == ST_RUN) {
                const u32 r = S.rem[jj] - J;
                S.rem[jj] = r;
                S.ctx[jj] += J;
                const i64 g0 = te0 - S.last[jj];  // first gap: from the slot's last token
                i64 mg = S.maxgap[jj];
                mg = g0 > mg ? g0 : mg;
                mg = tm1 > mg ? tm1 : mg;
                S.maxgap[jj] = mg;
                S.last[jj] = tend;
                fin = r == 0;
                if (fin)
                  write_record(rec + S.id[jj], S.ttft[jj], tend - S.arr[jj], mg, S.info[jj] >> 16,
                               TOKENSIM_REQ_FINISHED, (u32)klast);
                else
                  rmin_l = min(rmin_l, r);
              }
              u32 fm = __ballot_sync(FULLMASK, fin);
              __syncwarp();
              if (fm && first_fin == 0xffffffffu) first_fin = b0 + (u32)(__ffs(fm) - 1);
              nfin += __popc(fm);
              while (fm) {
                const u32 l = (u32)(__ffs(fm) - 1);
                fm &= fm - 1;
                const u32 pos = b0 + l;
                const u32 held = B.cdiv(S.ctx[pos]);
                const u32 slot = S.info[pos] & 0xffffu;
                free_blocks(S.bitmap, btD + (size_t)slot * btl, held, S.id[pos], klast, 2, L, hintD);
                nfreeD += held;
                if (lane == 0) atomicOr(&S.btfree[slot >> 5], 1u << (slot & 31u));
              }
            }
            __syncwarp();
            const u64 blkj = blk0 + Aj;
            it_reserve(L, 32);
            if (lj)
              it_put(L, lane, (kD + lane) | (1ull << 40), tsj, Tj, 0, Cdj, blkj, 0, nRun, 0, 0, 0,
                     lane == J - 1 ? nfin : 0u, 0);
            L.nit += J;
            nit += J;
            bnsD += warp_sum64(lj ? blkj * (u64)Tj : 0ull);
            trace_stretch(TA[1], FE[1], BINNED, FULLT, trcD, P.trace_cap, W, J, tsj, tej, blkj, flags);
            const u64 blk_last = blk0 + Ktot;
            peakD = blk_last > peakD ? blk_last : peakD;
            req_iters += (u64)nRun * J;
            if (nfin) {
              u32 out = first_fin;
              #pragma unroll 1
              for (u32 b0 = first_fin; b0 < nD; b0 += 32) {
                const u32 jj = b0 + lane;
                const bool valid = jj < nD;
                u32 vid = 0, vctx = 0, vrem = 0, vinfo = 0, vst = 0;
                i64 vl = 0, vm = 0, va = 0, vt = 0;
                if (valid) {
                  vid = S.id[jj];
                  vctx = S.ctx[jj];
                  vrem = S.rem[jj];
                  vinfo = S.info[jj];
                  vl = S.last[jj];
                  vm = S.maxgap[jj];
                  va = S.arr[jj];
                  vt = S.ttft[jj];
                  vst = stt[jj];
                }
                const bool keep = valid && vrem != 0;
                const u32 km = __ballot_sync(FULLMASK, keep);
                __syncwarp();
                if (keep) {
                  const u32 d = out + __popc(km & ltm);
                  S.id[d] = vid;
                  S.ctx[d] = vctx;
                  S.rem[d] = vrem;
                  S.info[d] = vinfo;
                  S.last[d] = vl;
                  S.maxgap[d] = vm;
                  S.arr[d] = va;
                  S.ttft[d] = vt;
                  stt[d] = vst;
                }
                __syncwarp();
                out += __popc(km);
              }
              nRun -= nfin;
              nD -= nfin;
              n_done += nfin;
              nfin_tot += nfin;
              last_fin = tend > last_fin ? tend : last_fin;
            }
            rminD = nRun ? __reduce_min_sync(FULLMASK, rmin_l) : 0u;
            ff_iters += J;
            ++ff_runs;
            tD = tend;
            lastD = tend;
            kD += J;
            D_idle = false;
            cyc_ffD += (u64)(prof_clock() - cD);
            continue;
          }
        }
        rminD = 0;
        const long long c1 = prof_clock();
        cyc_failD += (u64)(c1 - cD);
        cD = c1;
      }
      const u32 nA = nD - nX;  // running + preempted prefix
      // 3. decode reservation: RUN slots needing a block -> requester list (ascending id)
      u32 E = 0;
      u64 cdp = 0, npp = 0, app = 0;
      #pragma unroll 1
      for (u32 b0 = 0; b0 < nA; b0 += 32) {
        const u32 jj = b0 + lane;
        const bool run = jj < nA && stt[jj] == ST_RUN;
        const u32 c = run ? S.ctx[jj] : 1u;
        const bool need = run && B.mod(c) == 0;
        if (run) cdp += c + 1;
        const u32 bal = __ballot_sync(FULLMASK, need);
        if (need) {
          const u32 e = E + __popc(bal & ltm);
          S.req_cum[e] = e + 1;
          S.req_pt[e] = jj | (B.div(c) << 15);
        }
        E += __popc(bal);
      }
      u32 m = 0;
      u64 swap_out = 0;
      if ((u64)E > nfreeD) {
        // minimal m over the running slots, latest ids first; on D it may be all of them because
        // in-flight transfers hold unpreemptible blocks (reading R-PD4)
        u64 Sn = E, Hh = 0;
        u32 pos = nA;
        do {
          do {
            --pos;
          } while (stt[pos] != ST_RUN);
          ++m;
          const u32 c = S.ctx[pos];
          Sn -= (B.mod(c) == 0) ? 1 : 0;
          Hh += B.cdiv(c);
        } while (Sn > nfreeD + Hh && m < nRun);
        u64 csub = 0;
        u32 vpos = nA, done_v = 0;
        while (done_v < m) {
          do {
            --vpos;
          } while (stt[vpos] != ST_RUN);
          const u32 c = S.ctx[vpos];
          const u32 held = B.cdiv(c);
          free_blocks(S.bitmap, btD + (size_t)(S.info[vpos] & 0xffffu) * btl, held, S.id[vpos], kD, 2, L, hintD);
          nfreeD += held;
          csub += c + 1;
          if (SWAPM) swap_out += (u64)held * HPD.block_bytes;
          __syncwarp();
          if (lane == 0) {
            S.info[vpos] += 1u << 16;
            if (!SWAPM) S.ctx[vpos] = 0;
            stt[vpos] = ST_QUEUED;
          }
          __syncwarp();
          ++done_v;
        }
        if (lane == 0) cdp -= csub;
        E = (u32)Sn;
        nRun -= m;
        nQ += m;
        npre += m;
      }
      u32 Kb = E;
      nfreeD -= E;
      u32 nres = 0, nadm = 0, nrecomp = 0;
      u64 swap_in = 0, tokens = nRun;
      if (m == 0) {
        // 4. resume preempted requests in ascending id; |R| counts in-flight transfers too
        if (nQ > 0) {
          u64 cum_need = 0, cum_tok = 0;
          u32 taken = 0;
          #pragma unroll 1
          for (u32 b0 = 0; b0 < nA; b0 += 32) {
            const u32 jj = b0 + lane;
            const bool q = jj < nA && stt[jj] == ST_QUEUED;
            u32 need = 0, tok = 0, held0 = 0, c = 0;
            if (q) {
              if (SWAPM) {
                c = S.ctx[jj];
                need = B.cdiv(c) + (B.mod(c) == 0 ? 1u : 0u);
                tok = 1;
                held0 = B.cdiv(c);
              } else {
                const u32 id = S.id[jj];
                tok = PR[id] + (OU[id] - S.rem[jj]);
                need = B.cdiv(tok);
              }
            }
            const u32 qm = __ballot_sync(FULLMASK, q);
            const u32 rq = __popc(qm & ltm);
            const u32 cn = scan_incl(need), ct = scan_incl(tok);
            const bool ok = q && ((u64)nRun + nX + taken + rq + 1 <= (u64)mns) &&
                            (tokens + cum_tok + ct <= (u64)mbt) && ((i64)nfreeD - (i64)(cum_need + cn) >= wm);
            const u32 failm = __ballot_sync(FULLMASK, q && !ok);
            const u32 stopl = failm ? (u32)(__ffs(failm) - 1) : 32u;
            const bool take = q && lane < stopl;
            const u32 tm = __ballot_sync(FULLMASK, take);
            const u32 cnt = __popc(tm);
            if (take) {
              S.req_cum[E + rq] = Kb + cn;
              S.req_pt[E + rq] = jj;
              if (SWAPM) {
                stt[jj] = ST_RUN;
                cdp += c + 1;
              } else {
                stt[jj] = ST_RUN_RECOMP;
                S.ctx[jj] = tok;
                npp += tok;
                app += (u64)tok * (tok + 1) / 2;
              }
            }
            const u64 sw = warp_sum64(take ? (u64)held0 : 0ull);
            if (cnt) {
              const u32 last = 31u - __clz(tm);
              const u32 sn = __shfl_sync(FULLMASK, cn, last), stk = __shfl_sync(FULLMASK, ct, last);
              cum_need += sn;
              cum_tok += stk;
              Kb += sn;
              E += cnt;
              nres += cnt;
              taken += cnt;
              if (SWAPM) swap_in += sw * HPD.block_bytes;
              else nrecomp += cnt;
            }
            if (failm) break;
          }
          nfreeD -= cum_need;
          tokens += cum_tok;
          nRun += nres;
          nQ -= nres;
          __syncwarp();
        }
        // 5. pull visible pending requests FCFS and start their transfers (FIFO link)
        if (nQ == 0 && (!STATICP || (nRun == 0 && nX == 0))) {
          while (fdadm < ftail) {
            const u32 idx = fdadm + lane;
            const bool valid = idx < ftail;
            u32 id = 0, p = 0, o = 0;
            i64 join = INF, a = 0;
            if (valid) {
              id = fifo[idx].id;
              join = fifo[idx].join;
            }
            const bool vis = valid && join <= t;
            if (vis) {
              p = PR[id];
              o = OU[id];
              a = A[id];
            }
            const u32 need = B.cdiv(p);
            const u32 cneed = scan_incl(vis ? need : 0u);
            const bool ok = vis && ((u64)nRun + nX + lane + 1 <= (u64)mns) && ((i64)nfreeD - (i64)cneed >= wm);
            const u32 okm = __ballot_sync(FULLMASK, ok);
            const u32 cnt = (~okm == 0u) ? 32u : (u32)(__ffs(~okm) - 1);
            if (cnt == 0) break;
            const bool take = lane < cnt;
            const u32 slot = alloc_btslots(S.btfree, CAP / 32, take, lane, cnt);
            const i64 dur = take ? xfer_ns(p) : 0;
            const i64 start0 = t > link_busy ? t : link_busy;
            const i64 xend = start0 + scan_incl_i64(dur);
            if (take) {
              const u32 pos = nD + lane;
              S.id[pos] = id;
              S.ctx[pos] = p;
              S.rem[pos] = o - 1;
              S.info[pos] = slot;
              S.last[pos] = join;  // the first token left P at `join`
              S.maxgap[pos] = 0;
              S.arr[pos] = a;
              S.ttft[pos] = join - a;
              stt[pos] = ST_XFER;
              S.req_cum[E + lane] = Kb + cneed;
              S.req_pt[E + lane] = pos;
              fifo[idx].xend = xend;
            }
            const u32 sneed = __shfl_sync(FULLMASK, cneed, cnt - 1);
            const i64 x0 = __shfl_sync(FULLMASK, xend, 0);
            link_busy = __shfl_sync(FULLMASK, xend, cnt - 1);
            if (nX == 0) xhead_end = x0;
            if (fpfree >= fdadm && fpfree < fdadm + cnt) pf_end = __shfl_sync(FULLMASK, xend, fpfree - fdadm);
            if (P_idle && x0 < tP) tP = x0;  // P may be waiting for its blocks
            xbytes += warp_sum64(take ? (u64)p * P.M.kvb : 0ull);
            nfreeD -= sneed;
            Kb += sneed;
            E += cnt;
            nD += cnt;
            nX += cnt;
            fdadm += cnt;
            nadm += cnt;
            n_xfer += cnt;
            __syncwarp();
            if (cnt < 32) break;
          }
        }
      }
      if (Kb > 0 && !alloc_ordered(S, E, Kb, btD, btl, kD, 2, L, hintD, nwD)) {
        flags |= TOKENSIM_PT_INTERNAL_ERROR;
        break;
      }
      if (nRun == 0) {  // 6. nothing runnable: wake at the next transfer end or pending join
        if (fvis < fdadm) fvis = fdadm;
        while (fvis < ftail && fifo[fvis].join <= t) ++fvis;
        const i64 wj = fvis < ftail ? fifo[fvis].join : INF;
        tD = xhead_end < wj ? xhead_end : wj;
        D_idle = true;
        continue;
      }
      // 7. cost on D's profile
      const u32 Dn = nRun - nrecomp;
      const u64 Cd = warp_sum64(cdp);
      u64 Np = 0, Ap = 0;
      if (nrecomp) {
        Np = warp_sum64(npp);
        Ap = warp_sum64(app);
      }
      if (KD.preload && swap_in > 0) ev_flush(L);  // the event log doubles as the pipeline's scratch
      const i64 T = iter_time_chunk_ns(KD, Np, Ap, Np, nrecomp, Dn, Cd, swap_out, swap_in, reinterpret_cast<double *>(L.ev));
      const i64 te = t + T;
      const u64 blocks = totD - nfreeD;
      // 8. commit
      u32 nfin = 0, first_fin = 0xffffffffu, rmin_d = 0xffffffffu;
      #pragma unroll 1
      for (u32 b0 = 0; b0 < nA; b0 += 32) {
        const u32 jj = b0 + lane;
        bool fin = false;
        if (jj < nA) {
          const u32 st = stt[jj];
          if (st == ST_RUN || st == ST_RUN_RECOMP) {
            const u32 r = S.rem[jj] - 1;
            S.rem[jj] = r;
            if (st == ST_RUN) S.ctx[jj] += 1;
            else stt[jj] = ST_RUN;
            const i64 gap = te - S.last[jj];
            if (gap > S.maxgap[jj]) S.maxgap[jj] = gap;
            S.last[jj] = te;
            fin = r == 0;
            if (fin)
              write_record(rec + S.id[jj], S.ttft[jj], te - S.arr[jj], S.maxgap[jj], S.info[jj] >> 16,
                           TOKENSIM_REQ_FINISHED, (u32)kD);
            else
              rmin_d = min(rmin_d, r);
          }
        }
        u32 fm = __ballot_sync(FULLMASK, fin);
        __syncwarp();
        if (fm && first_fin == 0xffffffffu) first_fin = b0 + (u32)(__ffs(fm) - 1);
        nfin += __popc(fm);
        while (fm) {
          const u32 l = (u32)(__ffs(fm) - 1);
          fm &= fm - 1;
          const u32 pos = b0 + l;
          const u32 held = B.cdiv(S.ctx[pos]);
          const u32 slot = S.info[pos] & 0xffffu;
          free_blocks(S.bitmap, btD + (size_t)slot * btl, held, S.id[pos], kD, 2, L, hintD);
          nfreeD += held;
          if (lane == 0) atomicOr(&S.btfree[slot >> 5], 1u << (slot & 31u));
        }
      }
      __syncwarp();
      req_iters += nRun;
      if (nfin) {
        u32 out = first_fin;
        #pragma unroll 1
        for (u32 b0 = first_fin; b0 < nD; b0 += 32) {
          const u32 jj = b0 + lane;
          const bool valid = jj < nD;
          u32 vid = 0, vctx = 0, vrem = 0, vinfo = 0, vst = 0;
          i64 vl = 0, vm = 0, va = 0, vt = 0;
          if (valid) {
            vid = S.id[jj];
            vctx = S.ctx[jj];
            vrem = S.rem[jj];
            vinfo = S.info[jj];
            vl = S.last[jj];
            vm = S.maxgap[jj];
            va = S.arr[jj];
            vt = S.ttft[jj];
            vst = stt[jj];
          }
          const bool keep = valid && vrem != 0;
          const u32 km = __ballot_sync(FULLMASK, keep);
          __syncwarp();
          if (keep) {
            const u32 d = out + __popc(km & ltm);
            S.id[d] = vid;
            S.ctx[d] = vctx;
            S.rem[d] = vrem;
            S.info[d] = vinfo;
            S.last[d] = vl;
            S.maxgap[d] = vm;
            S.arr[d] = va;
            S.ttft[d] = vt;
            stt[d] = vst;
          }
          __syncwarp();
          out += __popc(km);
        }
        nRun -= nfin;
        nD -= nfin;
        n_done += nfin;
        nfin_tot += nfin;
        last_fin = te > last_fin ? te : last_fin;
      }
      rminD = __reduce_min_sync(FULLMASK, rmin_d);
      if (nRun == 0) rminD = 0;
      fold_iter(kD, 1, t, T, nrecomp, Dn, Np, Cd, m, nres, nadm, 0, nfin, blocks);
      trace_iter(TA[1], FE[1], BINNED, FULLT, trcD, P.trace_cap, W, t, te, blocks, flags);
      peakD = blocks > peakD ? blocks : peakD;
      bnsD += blocks * (u64)T;
      swo += swap_out;
      swi += swap_in;
      tD = te;
      lastD = te;
      ++kD;
      D_idle = false;
      cyc_normD += (u64)(prof_clock() - cD);
    } else {
      // ============================================================ P boundary
      const i64 t = tP;
      // P blocks of finished transfers come back (FIFO = transfer order)
      while (fpfree < fdadm && pf_end <= t) {
        const FifoEnt e = fifo[fpfree];
        u32 mn = 0xffffffffu;
        #pragma unroll 1
        for (u32 x0 = 0; x0 < e.len; x0 += 32) {
          ev_reserve(L, 32);
          const u32 x = x0 + lane;
          if (x < e.len) {
            const u32 b = ring[(e.seg + x) % ring_len];
            atomicOr(&bmP[b >> 5], 1u << (b & 31u));
            ev_put(L, x - x0, kP, 2, e.id, b);
            mn = min(mn, b >> 5);
          }
          L.nev += min(32u, e.len - x0);
        }
        mn = __reduce_min_sync(FULLMASK, mn);
        hintP = min(hintP, mn);
        nfreeP += e.len;
        ++fpfree;
        pf_end = fpfree < fdadm ? fifo[fpfree].xend : INF;
        __syncwarp();
      }
      while (arr < n) {
        if (arr >= win + 32) load_win(arr);
        const u32 mm = __ballot_sync(FULLMASK, (win + lane >= arr) && (wa <= t));
        arr += __popc(mm);
        if (arr < win + 32) break;
      }
      // fresh FCFS admission into a prefill batch
      u32 nb = 0, E = 0, Kb = 0, nrej = 0;
      u64 tokens = 0, npp = 0, app = 0;
      while (adm < arr) {
        const u32 i = adm + lane;
        const bool valid = i < arr;
        const u32 off = i - win;
        const bool inw = i >= win && off < 32;
        u32 p = __shfl_sync(FULLMASK, wp, off & 31u);
        u32 o = __shfl_sync(FULLMASK, wo, off & 31u);
        if (!valid) {
          p = 0;
          o = 0;
        } else if (!inw) {
          p = PR[i];
          o = OU[i];
        }
        const u32 need = B.cdiv(p);
        const bool rej = valid && (u64)need > HPP.cap_fresh;
        const bool el = valid && !rej;
        const u32 ce = scan_incl(el ? 1u : 0u);
        const u32 cneed = scan_incl(el ? need : 0u);
        const u32 cp = scan_incl(el ? p : 0u);
        const bool ok = el && ((u64)nb + ce <= (u64)mns) && (tokens + cp <= (u64)mbt) &&
                        ((i64)nfreeP - (i64)cneed >= wm);
        const u32 failm = __ballot_sync(FULLMASK, el && !ok);
        const u32 nvalid = min(32u, arr - adm);
        const u32 stop = failm ? (u32)(__ffs(failm) - 1) : nvalid;
        const bool take = el && lane < stop;
        const bool rj = rej && lane < stop;
        const u32 takem = __ballot_sync(FULLMASK, take);
        const u32 cnt = __popc(takem);
        if (take) {
          const u32 rank = __popc(takem & ltm);
          const u32 pos = nb + rank;
          pid[pos] = i;
          ppl[pos] = p;
          pol[pos] = o;
          S.req_cum[E + rank] = Kb + cneed;
          S.req_pt[E + rank] = pos;
          npp += p;
          app += (u64)p * (p + 1) / 2;
        }
        if (rj) reinterpret_cast<uint8_t *>(rec + i)[26] = (uint8_t)TOKENSIM_REQ_REJECTED;
        const u32 nrj = __popc(__ballot_sync(FULLMASK, rj));
        if (stop) {
          const u32 sneed = __shfl_sync(FULLMASK, cneed, stop - 1);
          const u32 sp = __shfl_sync(FULLMASK, cp, stop - 1);
          nfreeP -= sneed;
          Kb += sneed;
          tokens += sp;
        }
        E += cnt;
        nb += cnt;
        nrej += nrj;
        adm += stop;
        __syncwarp();
        if (stop < nvalid) break;
      }
      nrej_tot += nrej;
      n_done += nrej;
      if (nb == 0) {  // idle: wait for an arrival or for P blocks to come back
        const i64 wa_next = arr < n ? __shfl_sync(FULLMASK, wa, (arr - win) & 31u) : INF;
        tP = wa_next < pf_end ? wa_next : pf_end;
        P_idle = true;
        continue;
      }
      if (!alloc_ordered(SP, E, Kb, btP, btl, kP, 0, L, hintP, nwP)) {
        flags |= TOKENSIM_PT_INTERNAL_ERROR;
        break;
      }
      const u64 Np = warp_sum64(npp), Ap = warp_sum64(app);
      const i64 T = iter_time_ns(KP, Np, Ap, nb, 0, 0, 0);
      const i64 te = t + T;
      const u64 blocksP = totP - nfreeP;
      // commit: the first token; o == 1 finishes here, the rest join D's pending FIFO with
      // their P block lists moved into the ring
      u32 nfin = 0;
      #pragma unroll 1
      for (u32 b0 = 0; b0 < nb; b0 += 32) {
        const u32 pos = b0 + lane;
        const bool v = pos < nb;
        const u32 id = v ? pid[pos] : 0u, p = v ? ppl[pos] : 0u, o = v ? pol[pos] : 0u;
        const bool one = v && o == 1;
        const bool push = v && o > 1;
        const u32 need = B.cdiv(p);
        if (one) {
          const i64 a = A[id];
          write_record(rec + id, te - a, te - a, 0, 0, TOKENSIM_REQ_FINISHED, (u32)kP);
        }
        const u32 pm = __ballot_sync(FULLMASK, push);
        const u32 segx = scan_incl(push ? need : 0u) - (push ? need : 0u);
        const u32 rk = __popc(pm & ltm);
        if (push) {
          FifoEnt e;
          e.id = id;
          e.seg = (u32)((ring_tail + segx) % ring_len);
          e.len = need;
          e.pad = 0;
          e.join = te;
          e.xend = INF;
          fifo[ftail + rk] = e;
        }
        // move block lists (one request at a time, lanes over blocks) / free o == 1 blocks
        u32 vm = __ballot_sync(FULLMASK, v);
        while (vm) {
          const u32 l = (u32)(__ffs(vm) - 1);
          vm &= vm - 1;
          const u32 lpos = b0 + l;
          const u32 lneed = __shfl_sync(FULLMASK, need, l);
          const u32 lid = __shfl_sync(FULLMASK, id, l);
          const bool lone = __shfl_sync(FULLMASK, (u32)one, l) != 0u;
          const u32 lseg = __shfl_sync(FULLMASK, segx, l);
          const u32 *tbl = btP + (size_t)lpos * btl;
          if (lone) {
            free_blocks(bmP, tbl, lneed, lid, kP, 0, L, hintP);
            nfreeP += lneed;
          } else {
            #pragma unroll 1
            for (u32 x = lane; x < lneed; x += 32) ring[(ring_tail + lseg + x) % ring_len] = tbl[x];
          }
        }
        const u32 pushed_need = __shfl_sync(FULLMASK, scan_incl(push ? need : 0u), 31);
        ring_tail += pushed_need;
        ftail += __popc(pm);
        nfin += __popc(__ballot_sync(FULLMASK, one));
        __syncwarp();
      }
      n_done += nfin;
      nfin_tot += nfin;
      if (nfin) last_fin = te > last_fin ? te : last_fin;
      fold_iter(kP, 0, t, T, nb, 0, Np, 0, 0, 0, nb, nrej, nfin, blocksP);
      trace_iter(TA[0], FE[0], BINNED, FULLT, trcP, P.trace_cap, W, t, te, blocksP, flags);
      req_iters += nb;
      tP = te;
      lastP = te;
      ++kP;
      P_idle = false;
      if (D_idle && te < tD) tD = te;  // new pending requests join at te
    }
  }
  const i64 t_final = lastP > lastD ? lastP : lastD;
  if (BINNED) {
    for (int w = 0; w < 2; ++w)
      while ((i64)TA[w].bin * W < t_final) trace_flush_bin(TA[w], w ? trcD : trcP, P.trace_cap, W, flags);
  }
  // unfinished: D slots and requests still pending at D carry their first-token latency
  #pragma unroll 1
  for (u32 x = lane; x < nD; x += 32)
    write_record(rec + S.id[x], S.ttft[x], 0, 0, S.info[x] >> 16, TOKENSIM_REQ_UNFINISHED, 0);
  #pragma unroll 1
  for (u32 x = fdadm + lane; x < ftail; x += 32) {
    const u32 id = fifo[x].id;
    write_record(rec + id, fifo[x].join - A[id], 0, 0, 0, TOKENSIM_REQ_UNFINISHED, 0);
  }
  ev_flush(L);
  it_flush(L);
  const u64 dig_s = warp_sum64(L.dig_s);
  const u64 dig_b = warp_sum64(L.dig_b);
  if (lane == 0) {
    SimStats st;
    st.flags = flags | ((nrej_tot == n) ? (u32)TOKENSIM_PT_ALL_REJECTED : 0u);
    st.pad = 0;
    st.n_finished = nfin_tot;
    st.n_rejected = nrej_tot;
    st.n_iterations = kP + kD;
    st.n_req_iters = req_iters;
    st.n_preempt = npre;
    st.swap_out = swo;
    st.swap_in = swi;
    st.last_finish = last_fin;
    st.t_final = t_final;
    st.sched_d = dig_s;
    st.block_d = dig_b;
    st.req_d = 0;  // computed from the records by summary_kernel
    st.total_blocks = totD;
    st.peak_blocks = peakD;
    st.block_ns_sum = bnsD;
    st.trace_n[0] = FULLT ? FE[0].n : min(TA[0].tn, P.trace_cap);
    st.trace_n[1] = FULLT ? FE[1].n : min(TA[1].tn, P.trace_cap);
    for (int q = 2; q < 8; ++q) st.trace_n[q] = 0;
    st.trace_b[0] = FE[0].bytes;
    st.trace_b[1] = FE[1].bytes;
    for (int q = 2; q < 8; ++q) st.trace_b[q] = 0;
    st.iter_n = min(nit, P.it_cap);
    st.n_transfers = n_xfer;
    st.transfer_bytes = xbytes;
    st.ff_iters = ff_iters;
    st.ff_runs = ff_runs;
    st.cycles = (u64)(clock64() - clk0);
    st.cyc_ff = cyc_ffD;        // D: fast-forward stretches
    st.cyc_ff_fail = cyc_failD;  // D: attempts that did not run
    st.cyc_normal = cyc_normD;   // D: normal iterations (the rest: P, dispatch, idle D boundaries)
    for (int q = 0; q < 8; ++q) st.phase[q] = 0;
    for (int q = 0; q < 8; ++q) st.nphase[q] = 0;
    st.n_req = P.n_req;
    for (int q = 0; q < 5; ++q) st.ff_fail[q] = 0;
    for (int q = 0; q < 5; ++q) st.ff_cut[q] = 0;
    P.stats[j] = st;
  }
  __syncwarp();
}
