// sim_pdn.cuh -- NEXT-1: the xP:yD disaggregated node with a global scheduler (SURVEY §8(f)
// NEXT-1; readings R-X1..R-X6 in DESIGN.md).  Included by sim_core.cuh after sim_pd.cuh, inside
// namespace ts.  One CTA simulates one (prefill profile, decode profile) point: warp j runs
// decode worker j, and warp 0 also runs the global scheduler and the prefill workers -- or, in
// the SW build (one point per SM), warp y runs them on its own.
//
// x prefill workers and y decode workers run the a.9 worker loops; the
// global scheduler dispatches every arrival to a prefill worker and,
// at the end-of-prefill breakpoint, every request to a decode worker: round robin, least
// outstanding requests, or least allocated blocks, ties to the lowest index.  Dispatch events at
// time t run before worker boundaries at t, in request-id order; boundaries at equal times go
// decode workers first, then prefill workers, lower index first.  Each decode worker pulls its
// pending FIFO onto its own ingress link.
//
// Parallel decode workers (conservative epochs).  Decode workers interact with the rest of the
// node only through dispatches to them (which read their state) and through their pulls (which
// release prefill blocks at the transfer end).  The scheduler warp computes an epoch horizon H no
// dispatch can precede: the next known end-of-prefill dispatch, and -- since a prefill batch
// dispatches no earlier than one minimal prefill iteration (Tlb) after it starts -- the next
// arrival + Tlb, the next boundary + Tlb of a prefill worker with queued requests (one with an
// empty queue starts a batch only after an arrival), and (while a prefill worker is idle with
// queued requests, which a pull's block release could wake) the next decode boundary + Tlb.
// Then (1) every decode warp processes its own boundaries before H in parallel (quiet stretches
// cut at H), and (2) warp 0 processes the arrivals and prefill boundaries before H in time order
// and the dispatch events at H.  Decode boundaries precede prefill boundaries at equal times and
// dispatches precede boundaries at equal times, as in the sequential order; a pull that happens
// after a prefill boundary in time but before it in processing only lowers that worker's
// holder minimum, which the boundary recomputes from the same transfer ends (R-X6), so the
// result is the sequential one byte for byte (the node parity tests compare against the oracle's
// sequential loop).
//
// SW build: (2) runs alongside (1) on the scheduler's own warp.  Before a scheduler event at t it
// waits only for decode warps that could still pull before t (each publishes its next boundary
// and its unpulled FIFO entries after every boundary); pulls reach the prefill workers through
// per-worker mailboxes (atomicMin of the transfer end) that the scheduler folds before it looks
// at a prefill worker; and once every remaining request is with the decode workers it waits for
// all of them, so that it stops at the sequential loop's last event (E*).
//
// Data: per-worker scalars live in shared memory; decode worker j owns an id-sorted slot array +
// bitmap + its own requester lists in shared memory exactly like the pair's D; prefill workers own
// a bitmap each and share one batch table.  Per CTA in global memory: the decode FIFOs, the
// prefill queues / in-flight batches / holder lists, and per-request transfer ends and prefill
// block lists (a prefill worker frees a holder's blocks at its first boundary >= that holder's
// transfer end, in any order).

#pragma once
// (included inside namespace ts)

constexpr u32 PDN_MAXW = 8;

struct DScal {  // one decode worker
  i64 t, link_busy, xhead_end, last;
  u64 k, nfree, ffw, ffk, peak, bns;
  u32 hint, nD, nX, nQ, nRun, rmin, fhead, ftail, idle, pad;
  TraceAcc TA;
};
struct PScal {  // one prefill worker
  i64 t, tdisp, last, hmin;
  u64 k, nfree;
  u32 hint, qhead, qtail, nb, cur, nhold, idle, pad;
  TraceAcc TA;
};
struct PdnPart {  // one warp's partial outputs (summed by warp 0 at the end)
  u64 req_iters, npre, swo, swi, nfin, n_xfer, xbytes, ff_iters, ff_runs, dig_s, dig_b;
  i64 last_fin;
  i64 tfin;         // start of the latest iteration in which its decode worker finished requests
  u64 dcyc;         // SM cycles in decode phases (profile)
  u32 flags, done;  // done: requests its decode worker finished (read by warp 0 every epoch)
  FullEnc fe;       // its decode worker's FULL trace stream state
  i64 prog;         // SW: published during a phase -- every boundary before prog is processed
  u32 pend, pad2;   // SW: published during a phase -- FIFO entries not yet pulled
};
struct PdnCtl {
  i64 H;
  u32 stop, itcur;   // itcur: next free iteration-record position (warps flush in any order)
  i64 mb[PDN_MAXW];  // SW: per prefill worker, the earliest transfer end its holders' pulls set
                     // since the scheduler warp last looked (decode warps atomicMin, it exchanges)
};

struct PdnSmem {
  u32 *req_cum, *req_pt, *scratch, *pid, *ppl, *pol, *pinfo;
  PScal *ps;
  DScal *ds;
  u32 *bmP;              // [x][nwmax]
  unsigned char *dbase;  // decode worker j at dbase + j * dstride
  size_t dstride;
  u32 *dscr;             // decode warp j's requester lists at dscr + j * (2 cap + 64)
  PdnPart *part;         // [y + 1]: the decode warps, then (SW) the scheduler warp
  PdnCtl *ctl;
  CostK *kc;             // [2]: the prefill and decode profiles' cost constants
};

__host__ __device__ inline size_t pdn_dworker_bytes(u32 cap, u32 nw) {
  return ((size_t)cap * (8 * 4 + 4 * 5) + (size_t)(cap / 32) * 4 + (size_t)nw * 4 + 15) & ~(size_t)15;
}
__host__ __device__ inline size_t pdn_base_bytes(u32 cap, u32 nw, u32 x, u32 y) {
  size_t b = (size_t)cap * 4 * 6 + 64 * 4;
  b = (b + 15) & ~(size_t)15;
  b += (size_t)x * sizeof(PScal) + (size_t)y * sizeof(DScal);
  b = (b + 15) & ~(size_t)15;
  b += ((size_t)x * nw * 4 + 15) & ~(size_t)15;
  b += (size_t)y * pdn_dworker_bytes(cap, nw);
  return b;
}
// shared memory of one node CTA (one point)
__host__ __device__ inline size_t pdn_smem_per_warp(u32 cap, u32 nw, u32 x, u32 y) {
  size_t b = pdn_base_bytes(cap, nw, x, y);
  b += (size_t)y * ((size_t)cap * 8 + 64 * 4);
  b = (b + 15) & ~(size_t)15;
  b += (size_t)(y + 1) * sizeof(PdnPart);
  b = (b + 15) & ~(size_t)15;
  b += (sizeof(PdnCtl) + 15) & ~(size_t)15;
  b += (2 * sizeof(CostK) + 15) & ~(size_t)15;
  return b;
}

__device__ __forceinline__ PdnSmem carve_pdn(unsigned char *base, u32 cap, u32 nw, u32 x, u32 y) {
  PdnSmem M;
  u32 *p32 = reinterpret_cast<u32 *>(base);
  M.req_cum = p32;
  M.req_pt = p32 + cap;
  M.pid = p32 + 2 * cap;
  M.ppl = p32 + 3 * cap;
  M.pol = p32 + 4 * cap;
  M.pinfo = p32 + 5 * cap;
  M.scratch = p32 + 6 * cap;
  size_t o = ((size_t)cap * 4 * 6 + 64 * 4 + 15) & ~(size_t)15;
  M.ps = reinterpret_cast<PScal *>(base + o);
  o += (size_t)x * sizeof(PScal);
  M.ds = reinterpret_cast<DScal *>(base + o);
  o += (size_t)y * sizeof(DScal);
  o = (o + 15) & ~(size_t)15;
  M.bmP = reinterpret_cast<u32 *>(base + o);
  o += ((size_t)x * nw * 4 + 15) & ~(size_t)15;
  M.dbase = base + o;
  M.dstride = pdn_dworker_bytes(cap, nw);
  o += (size_t)y * M.dstride;
  M.dscr = reinterpret_cast<u32 *>(base + o);
  o += (size_t)y * ((size_t)cap * 8 + 64 * 4);
  o = (o + 15) & ~(size_t)15;
  M.part = reinterpret_cast<PdnPart *>(base + o);
  o += (size_t)(y + 1) * sizeof(PdnPart);
  o = (o + 15) & ~(size_t)15;
  M.ctl = reinterpret_cast<PdnCtl *>(base + o);
  o += (sizeof(PdnCtl) + 15) & ~(size_t)15;
  M.kc = reinterpret_cast<CostK *>(base + o);
  return M;
}

// the WarpSmem view of decode worker j (slots, bitmap) plus its own requester lists
__device__ __forceinline__ WarpSmem dview(const PdnSmem &M, u32 j, u32 cap, u32 **stt) {
  WarpSmem S;
  unsigned char *b = M.dbase + (size_t)j * M.dstride;
  i64 *p64 = reinterpret_cast<i64 *>(b);
  S.last = p64;
  S.maxgap = p64 + cap;
  S.arr = p64 + 2 * cap;
  S.ttft = p64 + 3 * cap;
  u32 *p32 = reinterpret_cast<u32 *>(p64 + 4 * cap);
  S.id = p32;
  S.ctx = p32 + cap;
  S.rem = p32 + 2 * cap;
  S.info = p32 + 3 * cap;
  *stt = p32 + 4 * cap;
  S.btfree = p32 + 5 * cap;
  S.bitmap = p32 + 5 * cap + cap / 32;
  u32 *sc = M.dscr + (size_t)j * (2 * cap + 64);
  S.req_cum = sc;
  S.req_pt = sc + cap;
  S.scratch = sc + 2 * cap;
  return S;
}

// argmin of key over lanes 0..7 (a node has at most 8 workers; lane = worker order), ties to
// the lower lane; three butterfly steps within each group of 8 lanes, then lane 0's answer
__device__ __forceinline__ u32 warp_argmin64(i64 key, bool valid) {
  i64 k = valid ? key : INT64_MAX;
  u32 who = valid ? lane_id() : 0xffffffffu;
#pragma unroll
  for (u32 s = 4; s; s >>= 1) {
    const i64 k2 = __shfl_xor_sync(FULLMASK, k, s);
    const u32 w2 = __shfl_xor_sync(FULLMASK, who, s);
    if (k2 < k || (k2 == k && w2 < who)) {
      k = k2;
      who = w2;
    }
  }
  return __shfl_sync(FULLMASK, who, 0);
}
// min over lanes 0..7 (the other lanes hold no worker), broadcast to the warp
__device__ __forceinline__ i64 min8_i64(i64 x) {
#pragma unroll
  for (u32 s = 4; s; s >>= 1) {
    const i64 y = __shfl_xor_sync(FULLMASK, x, s);
    x = y < x ? y : x;
  }
  return __shfl_sync(FULLMASK, x, 0);
}
__device__ __forceinline__ i64 sat_add(i64 a, i64 b) { return a >= INT64_MAX - b ? INT64_MAX : a + b; }

// iteration log of one warp of a node CTA: its records go to positions claimed from the CTA's
// shared cursor (the warps flush in any order; node records are compared by (worker, k))
static __device__ __noinline__ void pdn_it_flush(Logs &L, u32 *itcur) {
  u32 base = 0;
  if (lane_id() == 0) base = atomicAdd(itcur, L.nit);
  L.it_base = __shfl_sync(FULLMASK, base, 0);
  it_flush(L);
}
__device__ __forceinline__ void pdn_it_reserve(Logs &L, u32 cnt, u32 *itcur) {
  if (L.nit + cnt > ITCAP) pdn_it_flush(L, itcur);
}

template <int CAP, bool P2, bool SW>
__device__ void simulate_pdn(const SweepParams &P, u64 j, unsigned char *smem, u32 *bt, u32 wib) {
  const u32 lane = lane_id();
  const u32 ltm = lanemask_lt();
  const u32 X = P.pd_x, Y = P.pd_y, NW = X + Y;
  // the scheduler warp: warp 0, which also runs decode worker 0, or (SW) warp y, a warp of its own
  const bool COORD = SW ? wib == P.pd_y : wib == 0;
  const u64 point = P.begin + j * P.stride;
  const Coords cd = decode_point(point, P.n_pol, P.n_rates, P.n_seeds);
  const u32 hwP = cd.hw / P.n_hw, hwD = cd.hw % P.n_hw;
  const DevHP HPP = P.hp[(size_t)hwP * P.n_pol + cd.pol];
  const DevHP HPD = P.hp[(size_t)hwD * P.n_pol + cd.pol];
  const DevPol PL = P.pol[cd.pol];
  const PdnSmem M = carve_pdn(smem, CAP, P.nwords_max, X, Y);
  // the cost constants live in shared memory (read at each use: registers stay free for the
  // chain's state -- the two-CTAs-per-SM build caps them at 168)
  if (threadIdx.x == 0) {
    M.kc[0] = make_costk(P.M, P.MF, P.hw[hwP]);
    M.kc[1] = make_costk(P.M, P.MF, P.hw[hwD], P.link_mode, P.preload_buf);
  }
  __syncthreads();
  const CostK &KP = M.kc[0];
  const CostK &KD = M.kc[1];
  const u32 g = P.group_of_point_mode ? 0u : cd.rate * P.n_seeds + cd.seed;
  const u32 n = P.n_req;
  const i64 *A = P.arrival + (size_t)g * n;
  const u32 *PR = P.prompt + (size_t)g * n;
  const u32 *OU = P.output + (size_t)g * n;
  tokensim_request_record *rec = P.rec + (size_t)j * n;
  tokensim_mem_sample *trc0 = P.trace + (size_t)j * P.trace_nw * P.trace_cap;
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
  const u32 gwarp = blockIdx.x * (Y + (SW ? 1u : 0u)) + wib;  // this warp's logs
  PdnCtl *ctl = M.ctl;
  u32 *itcur = &ctl->itcur;
  // per-CTA global scratch
  unsigned char *gb = P.pdn_scratch + (size_t)blockIdx.x * P.pdn_bytes_per_warp;
  FifoEnt *fifo0 = reinterpret_cast<FifoEnt *>(gb);                  // [y][n]
  u32 *qP0 = reinterpret_cast<u32 *>(fifo0 + (size_t)Y * n);         // [x][n] dispatch queues
  u32 *hold0 = qP0 + (size_t)X * n;                                  // [x][n] holder lists
  u32 *batch0 = hold0 + (size_t)X * n;                               // [x][CAP] in-flight batches
  i64 *reqx = reinterpret_cast<i64 *>((reinterpret_cast<uintptr_t>(batch0 + (size_t)X * CAP) + 7) & ~(uintptr_t)7);
  u32 *pblk = reinterpret_cast<u32 *>(reqx + n);                     // [n][btl] prefill block lists
  u32 *btD0 = bt;                                                    // [y][CAP][btl]
  u32 *btP = bt + (size_t)Y * CAP * btl;                             // shared prefill batch table
  WarpSmem SP;  // the prefill batch view for the allocator (warp 0)
  SP.id = M.pid;
  SP.info = M.pinfo;
  SP.req_cum = M.req_cum;
  SP.req_pt = M.req_pt;
  SP.scratch = M.scratch;
  const TraceAcc ta0 = {0, 0, 0, (i64)P.bin_ns, 0, 0};
  // this warp's decode worker
  const u32 dj = (SW && COORD) ? 0u : wib;  // (the SW scheduler warp's views are never used)
  const u32 wid = X + dj;
  const u32 koffD = 2 * wid;
  u32 *stt;
  const WarpSmem S = dview(M, dj, CAP, &stt);
  FifoEnt *fifo = fifo0 + (size_t)dj * n;
  u32 *btD = btD0 + (size_t)dj * CAP * btl;
  tokensim_mem_sample *trcD = trc0 + (size_t)wid * P.trace_cap;

  // ---- init (every warp: its decode worker; warp 0: the prefill workers and the controls)
  {
    const u32 tid = threadIdx.x, nth = blockDim.x;
    ulonglong2 *r2 = reinterpret_cast<ulonglong2 *>(rec);
    const ulonglong2 z = make_ulonglong2(0ull, 0ull);
    #pragma unroll 1
    for (u32 x = tid; x < 2 * n; x += nth) r2[x] = z;
    #pragma unroll 1
    for (u32 x = tid; x < n; x += nth) reqx[x] = INF;
    const bool has_d = !(SW && COORD);  // (the SW scheduler warp runs no decode worker)
    if (has_d) {
      const u32 fw = (u32)(totD >> 5), tl = (u32)(totD & 31u);
      #pragma unroll 1
      for (u32 q = lane; q < nwD; q += 32) S.bitmap[q] = q < fw ? 0xffffffffu : (q == fw && tl ? ((1u << tl) - 1u) : 0u);
      #pragma unroll 1
      for (u32 q = lane; q < CAP / 32; q += 32) S.btfree[q] = 0xffffffffu;
    }
    if (lane == 0 && has_d) {
      DScal s;
      s.t = INF;  // a decode worker starts idle: a dispatch wakes it
      s.link_busy = 0;
      s.xhead_end = INF;
      s.last = 0;
      s.k = 0;
      s.nfree = totD;
      s.ffw = s.ffk = s.peak = s.bns = 0;
      s.hint = 0;
      s.nD = s.nX = s.nQ = s.nRun = s.rmin = s.fhead = s.ftail = 0;
      s.idle = 1;
      s.pad = 0;
      s.TA = ta0;
      M.ds[dj] = s;
    }
    if (lane == 0) {
      M.part[wib].done = 0;
      M.part[wib].flags = 0;
    }
    if (COORD) {
      for (u32 w = 0; w < X; ++w) {
        u32 *bm = M.bmP + (size_t)w * P.nwords_max;
        const u32 fw = (u32)(totP >> 5), tl = (u32)(totP & 31u);
        #pragma unroll 1
        for (u32 q = lane; q < nwP; q += 32) bm[q] = q < fw ? 0xffffffffu : (q == fw && tl ? ((1u << tl) - 1u) : 0u);
      }
      #pragma unroll 1
      for (u32 x = lane; x < CAP; x += 32) M.pinfo[x] = x;
      if (lane == 0) {
        for (u32 w = 0; w < X; ++w) {
          PScal s;
          s.t = INF;  // a prefill worker starts idle: a dispatch wakes it
          s.tdisp = INF;
          s.last = 0;
          s.hmin = INF;
          s.k = 0;
          s.nfree = totP;
          s.hint = 0;
          s.qhead = s.qtail = s.nb = s.cur = s.nhold = 0;
          s.idle = 1;
          s.pad = 0;
          s.TA = ta0;
          M.ps[w] = s;
        }
        ctl->itcur = 0;
        ctl->stop = 0;
        ctl->H = INF;
        for (u32 w = 0; w < PDN_MAXW; ++w) ctl->mb[w] = INF;
      }
    }
    __syncthreads();
  }
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
  // this warp's partial outputs
  u64 req_iters = 0, npre = 0, swo = 0, swi = 0, nfin_tot = 0, n_xfer = 0, xbytes = 0;
  u64 ff_iters = 0, ff_runs = 0;
  u32 flags = 0, done_w = 0;
  i64 last_fin = 0, tfin_w = 0;
  // warp 0 only: the scheduler's state
  u32 arr = 0, n_done_c = 0, n_toD = 0;  // n_toD: requests dispatched to decode workers
  // A[arr], A[arr + 1] and PR[arr] kept in registers (their loads leave the chain)
  i64 ta_next = n > 0 ? A[0] : INT64_MAX;
  i64 ta_next2 = n > 1 ? A[1] : INT64_MAX;
  u32 pr_next = n > 0 ? PR[0] : 0u;
  auto advance_arr = [&]() {
    ++arr;
    ta_next = ta_next2;
    ta_next2 = arr + 1 < n ? A[arr + 1] : INT64_MAX;
    pr_next = arr < n ? PR[arr] : 0u;
  };
  u64 rrP = 0, rrD = 0, nrej_tot = 0;
  const bool ff_on = P.ff_enable != 0;
  const bool BINNED = P.trace_mode == TOKENSIM_TRACE_BINNED;
  const bool FULLT = P.trace_mode == TOKENSIM_TRACE_FULL;
  const i64 W = (i64)P.bin_ns;
  FullEnc fe = {0, 0, 0, 0, 0, 0};  // this warp's decode worker's FULL stream (lane-uniform)
  FullEnc FEp[PDN_MAXW];            // warp 0: the prefill workers' streams
  for (u32 w = 0; w < PDN_MAXW; ++w) FEp[w] = {0, 0, 0, 0, 0, 0};
  // a prefill batch takes at least one minimal prefill iteration (1 prompt of 1 token; every
  // c.5 term grows with the batch), less a margin for rounding: dispatches come >= Tlb after a
  // batch starts
  i64 Tlb;
  {
    const i64 t1 = iter_time_ns(KP, 1, 1, 1, 0, 0, 0);
    Tlb = t1 - (t1 >> 6) - 1;
    if (Tlb < 1) Tlb = 1;
  }
  auto fold_iter = [&](u64 kk, u32 worker, i64 ts, i64 T, u64 Sp, u64 D_, u64 Np, u64 Cd, u64 m, u64 nres,
                       u64 nadm, u64 nrej, u64 nfin, u64 blocks) {
    pdn_it_reserve(L, 1, itcur);
    if (lane == 0) it_put(L, 0, kk | ((u64)worker << 40), ts, T, Np, Cd, blocks, Sp, D_, m, nres, nadm, nfin, nrej);
    L.nit += 1;
  };
  auto xfer_ns = [&](u32 p) -> i64 {
    const u64 bytes = (u64)p * P.M.kvb;
    return (i64)floor(__dadd_rn(__dmul_rn(__dmul_rn(__ull2double_rn(bytes), P.pd_link_inv), 1e9), 0.5));
  };
  // global scheduler (reading R-X2): round robin, or the argmin of outstanding requests /
  // allocated blocks as of each worker's last processed boundary; ties to the lowest index
  auto pick = [&](bool toD, i64 tnow) -> u32 {
    const u32 cnt = toD ? Y : X;
    if (P.dispatch == TOKENSIM_DISPATCH_ROUND_ROBIN) return (u32)((toD ? rrD++ : rrP++) % cnt);
    u64 v = ~0ull;
    if (lane < cnt) {
      if (P.dispatch == TOKENSIM_DISPATCH_LEAST_OUTSTANDING) {
        if (toD) {
          const DScal &d = M.ds[lane];
          v = (u64)(d.ftail - d.fhead) + d.nD;
        } else {
          const PScal &p = M.ps[lane];
          v = (u64)(p.qtail - p.qhead) + (p.tdisp == tnow ? 0u : p.nb);  // batches completing now are gone
        }
      } else {
        v = toD ? totD - M.ds[lane].nfree : totP - M.ps[lane].nfree;
      }
    }
    const u32 w = warp_argmin64((i64)v, lane < cnt);
    return w;
  };

  // one boundary of this warp's decode worker (the D_j boundary of the sequential loop) before
  // the epoch horizon H; false on an internal error
  DScal d;  // this warp's decode worker's scalars, in registers while a phase runs
  auto d_step = [&](const i64 H) -> bool {
    const u32 koff = koffD;
    const i64 t = d.t;
    // 1. finished transfers become runnable (the in-flight tail completes in FIFO order)
    // (transfers on this worker's link end in pull order; slots are id-sorted, so find by id)
    while (d.nX > 0 && d.xhead_end <= t) {
      const u32 xid = fifo[d.fhead - d.nX].id;
      #pragma unroll 1
      for (u32 b0 = 0; b0 < d.nD; b0 += 32) {
        const u32 jj = b0 + lane;
        const u32 hit = __ballot_sync(FULLMASK, jj < d.nD && S.id[jj] == xid);
        if (hit) {
          if (lane == 0) stt[b0 + (u32)(__ffs(hit) - 1)] = ST_RUN;
          break;
        }
      }
      --d.nX;
      ++d.nRun;
      d.xhead_end = d.nX ? fifo[d.fhead - d.nX].xend : INF;
    }
    __syncwarp();
    bool ff_done = false;
    // ---------------------------------------------------------- D fast-forward (H3)
    // Quiescent decode stretch: no transfer completes, nothing is pulled or resumed, nothing
    // is preempted, and no dispatch (which reads this worker's state or feeds its FIFO) can
    // happen before the stretch's iterations: every iteration starts before the epoch
    // horizon H, which no dispatch precedes.
    if (ff_on && d.nRun > 0 && d.rmin >= 2 && (d.nfree > d.ffw || d.k >= d.ffk)) {
      const i64 cut = H - 1;  // iterations starting at or after the epoch horizon H are excluded
      bool quiet = true, mem_check = false;
      u32 need_h = 0;
      const u32 nA0 = d.nD;  // all slots (states are checked)
      if (d.nQ > 0) {
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
        if (!((u64)d.nRun + d.nX + 1 > mns || (u64)d.nRun + tokq > mbt)) {
          mem_check = true;
          if ((i64)d.nfree - (i64)d.nRun - (i64)need_h >= wm) quiet = false;
        }
      } else if (!STATICP && d.fhead < d.ftail) {
        // a visible pending head (every FIFO entry is visible): blocked now => blocked later
        need_h = B.cdiv(PR[fifo[d.fhead].id]);
        if (!((u64)d.nRun + d.nX + 1 > mns)) {
          mem_check = true;
          if ((i64)d.nfree - (i64)d.nRun - (i64)need_h >= wm) quiet = false;
        }
      }
      if (quiet) {
        S.scratch[lane] = 0;
        S.scratch[32 + lane] = 0;
        __syncwarp();
        u64 cdp0 = 0;
        u32 rmn = 0xffffffffu;
        #pragma unroll 1
        for (u32 b0 = 0; b0 < nA0; b0 += 32) {
          const u32 jj = b0 + lane;
          u32 key = 64u + lane;
          if (jj < nA0 && stt[jj] == ST_RUN) {
            const u32 c = S.ctx[jj];
            cdp0 += c + 1;
            rmn = min(rmn, S.rem[jj]);
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
        const u32 nj = S.scratch[B.bs >= 32 ? lane : B.mod(lane)];
        const u32 Aj = scan_incl(nj);
        const u64 Cdj = Cd0 + (u64)lane * d.nRun;
        const i64 Tj = iter_time_ns(KD, 0, 0, 0, d.nRun, Cdj, 0);
        const i64 tej = t + scan_incl_i64(Tj);
        const i64 tsj = tej - Tj;
        bool ok = ((u64)Aj <= d.nfree) && (Aj <= (u32)CAP) && (lane < rm);
        if (lane > 0) {
          if (P.horizon >= 0 && tsj >= P.horizon) ok = false;
          if (tsj >= d.xhead_end || tsj > cut) ok = false;
        }
        if (mem_check) {
          const u64 fr = d.nfree - (u64)__shfl_sync(FULLMASK, Aj, 0);
          if (!((i64)fr - (i64)need_h < wm)) ok = false;
        }
        const u32 okm = __ballot_sync(FULLMASK, ok);
        const u32 J = (~okm == 0u) ? 32u : (u32)(__ffs(~okm) - 1);
        const u32 memcut = __ballot_sync(FULLMASK, !((u64)Aj <= d.nfree));
        if (J < 2 && memcut && (u32)(__ffs(memcut) - 1) < 2) {
          d.ffw = d.nfree;
          d.ffk = d.k + 4;
        }
        if (J >= 2) {
          const u32 Ktot = __shfl_sync(FULLMASK, Aj, J - 1);
          __syncwarp();
          S.scratch[lane] = Aj - nj;  // bucket cursors
          __syncwarp();
          if (Ktot > 0) {
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
            if (!alloc_ordered(S, Ktot, Ktot, btD, btl, d.k, koff, L, d.hint, nwD)) {
              flags |= TOKENSIM_PT_INTERNAL_ERROR;
              return false;
            }
          }
          const u64 blk0 = totD - d.nfree;
          d.nfree -= Ktot;
          const u64 klast = d.k + J - 1;
          const i64 tend = __shfl_sync(FULLMASK, tej, J - 1);
          const i64 te0 = __shfl_sync(FULLMASK, tej, 0);
          const bool lj = lane < J;
          i64 tm1 = (lj && lane > 0) ? Tj : 0;
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
              const i64 g0 = te0 - S.last[jj];
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
              const u32 slot = SLOT(S.info[pos]);
              free_blocks(S.bitmap, btD + (size_t)slot * btl, held, S.id[pos], klast, koff, L, d.hint);
              d.nfree += held;
              if (lane == 0) atomicOr(&S.btfree[slot >> 5], 1u << (slot & 31u));
            }
          }
          __syncwarp();
          const u64 blkj = blk0 + Aj;
          pdn_it_reserve(L, 32, itcur);
          if (lj)
            it_put(L, lane, (d.k + lane) | ((u64)wid << 40), tsj, Tj, 0, Cdj, blkj, 0, d.nRun, 0, 0, 0,
                   lane == J - 1 ? nfin : 0u, 0);
          L.nit += J;
          d.bns += warp_sum64(lj ? blkj * (u64)Tj : 0ull);
          trace_stretch(d.TA, fe, BINNED, FULLT, trcD, P.trace_cap, W, J, tsj, tej, blkj, flags);
          const u64 blk_last = blk0 + Ktot;
          d.peak = blk_last > d.peak ? blk_last : d.peak;
          req_iters += (u64)d.nRun * J;
          if (nfin) {
            u32 out = first_fin;
            #pragma unroll 1
            for (u32 b0 = first_fin; b0 < d.nD; b0 += 32) {
              const u32 jj = b0 + lane;
              const bool valid = jj < d.nD;
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
                const u32 dd = out + __popc(km & ltm);
                S.id[dd] = vid;
                S.ctx[dd] = vctx;
                S.rem[dd] = vrem;
                S.info[dd] = vinfo;
                S.last[dd] = vl;
                S.maxgap[dd] = vm;
                S.arr[dd] = va;
                S.ttft[dd] = vt;
                stt[dd] = vst;
              }
              __syncwarp();
              out += __popc(km);
            }
            d.nRun -= nfin;
            d.nD -= nfin;
            done_w += nfin;
            nfin_tot += nfin;
            last_fin = tend > last_fin ? tend : last_fin;
            tfin_w = __shfl_sync(FULLMASK, tsj, J - 1);
          }
          d.rmin = d.nRun ? __reduce_min_sync(FULLMASK, rmin_l) : 0u;
          ff_iters += J;
          ++ff_runs;
          d.t = tend;
          d.last = tend;
          d.k += J;
          d.idle = 0;
          ff_done = true;
        }
      }
      if (!ff_done) d.rmin = 0;
    }
    if (flags & TOKENSIM_PT_INTERNAL_ERROR) return false;
    if (!ff_done) {
      const u32 nA = d.nD;  // all slots, id-sorted (states are checked)
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
      if ((u64)E > d.nfree) {
        // minimal m over the running slots, latest ids first (in-flight blocks are not preemptible)
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
        } while (Sn > d.nfree + Hh && m < d.nRun);
        u64 csub = 0;
        u32 vpos = nA, done_v = 0;
        while (done_v < m) {
          do {
            --vpos;
          } while (stt[vpos] != ST_RUN);
          const u32 c = S.ctx[vpos];
          const u32 held = B.cdiv(c);
          free_blocks(S.bitmap, btD + (size_t)SLOT(S.info[vpos]) * btl, held, S.id[vpos], d.k, koff, L, d.hint);
          d.nfree += held;
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
        d.nRun -= m;
        d.nQ += m;
        npre += m;
      }
      u32 Kb = E;
      d.nfree -= E;
      u32 nres = 0, nadm = 0, nrecomp = 0;
      u64 swap_in = 0, tokens = d.nRun;
      if (m == 0) {
        // 4. resume preempted requests in ascending id; |R| counts in-flight transfers too
        if (d.nQ > 0) {
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
            const bool ok = q && ((u64)d.nRun + d.nX + taken + rq + 1 <= (u64)mns) &&
                            (tokens + cum_tok + ct <= (u64)mbt) && ((i64)d.nfree - (i64)(cum_need + cn) >= wm);
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
          d.nfree -= cum_need;
          tokens += cum_tok;
          d.nRun += nres;
          d.nQ -= nres;
          __syncwarp();
        }
        // 5. pull pending requests FCFS and start their transfers on this worker's link
        if (d.nQ == 0 && (!STATICP || (d.nRun == 0 && d.nX == 0))) {
          while (d.fhead < d.ftail) {
            const u32 idx = d.fhead + lane;
            const bool valid = idx < d.ftail;
            u32 id = 0, p = 0, o = 0, pw = 0;
            i64 join = INF, a = 0;
            if (valid) {
              const FifoEnt e = fifo[idx];
              id = e.id;
              pw = e.seg;
              join = e.join;
            }
            const bool vis = valid && join <= t;
            if (vis) {
              p = PR[id];
              o = OU[id];
              a = A[id];
            }
            const u32 need = B.cdiv(p);
            const u32 cneed = scan_incl(vis ? need : 0u);
            const bool ok = vis && ((u64)d.nRun + d.nX + lane + 1 <= (u64)mns) && ((i64)d.nfree - (i64)cneed >= wm);
            const u32 okm = __ballot_sync(FULLMASK, ok);
            const u32 cnt = (~okm == 0u) ? 32u : (u32)(__ffs(~okm) - 1);
            if (cnt == 0) break;
            const bool take = lane < cnt;
            const u32 slot = alloc_btslots(S.btfree, CAP / 32, take, lane, cnt);
            const i64 dur = take ? xfer_ns(p) : 0;
            const i64 start0 = t > d.link_busy ? t : d.link_busy;
            const i64 xend = start0 + scan_incl_i64(dur);
            if (take) {
              const u32 pos = d.nD + lane;
              S.id[pos] = id;
              S.ctx[pos] = p;
              S.rem[pos] = o - 1;
              S.info[pos] = slot;
              S.last[pos] = join;  // the first token left its prefill worker at `join`
              S.maxgap[pos] = 0;
              S.arr[pos] = a;
              S.ttft[pos] = join - a;
              stt[pos] = ST_XFER;
              S.req_cum[E + lane] = Kb + cneed;
              S.req_pt[E + lane] = pos;
              fifo[idx].xend = xend;
              reqx[id] = xend;
            }
            __syncwarp();
            if constexpr (SW) __threadfence_block();  // reqx before the mailbox (read concurrently)
            // the holders' prefill workers: their blocks come back at xend (wake idle ones)
            for (u32 l = 0; l < cnt; ++l) {
              const u32 lpw = __shfl_sync(FULLMASK, pw, l);
              const i64 lx = __shfl_sync(FULLMASK, xend, l);
              if (lane == 0) {  // several decode warps may release to one prefill worker at once
                if constexpr (SW) {  // the scheduler warp runs concurrently: through its mailbox
                  atomicMin(reinterpret_cast<long long *>(&ctl->mb[lpw]), (long long)lx);
                } else {
                  PScal &ps = M.ps[lpw];
                  atomicMin(reinterpret_cast<long long *>(&ps.hmin), (long long)lx);
                  if (ps.idle) atomicMin(reinterpret_cast<long long *>(&ps.t), (long long)lx);
                }
              }
            }
            __syncwarp();
            const u32 sneed = __shfl_sync(FULLMASK, cneed, cnt - 1);
            const i64 x0 = __shfl_sync(FULLMASK, xend, 0);
            d.link_busy = __shfl_sync(FULLMASK, xend, cnt - 1);
            if (d.nX == 0) d.xhead_end = x0;
            xbytes += warp_sum64(take ? (u64)p * P.M.kvb : 0ull);
            d.nfree -= sneed;
            Kb += sneed;
            E += cnt;
            d.nD += cnt;
            d.nX += cnt;
            d.fhead += cnt;
            nadm += cnt;
            n_xfer += cnt;
            __syncwarp();
            if (cnt < 32) break;
          }
        }
      }
      if (Kb > 0 && !alloc_ordered(S, E, Kb, btD, btl, d.k, koff, L, d.hint, nwD)) {
        flags |= TOKENSIM_PT_INTERNAL_ERROR;
        return false;
      }
      // pulled requests were appended in dispatch order, which with several prefill workers
      // need not be id order: insert them into the id-sorted slots (victims are the latest
      // arrivals, requesters go in id order -- reading A7).  In-flight slots cannot finish in
      // this iteration, so doing it before the commit keeps positions stable for it.
      for (u32 q = d.nD - nadm; q < d.nD; ++q) {
        const u32 qid = S.id[q];
        u32 p = 0;
        #pragma unroll 1
        for (u32 b0 = 0; b0 < q; b0 += 32) {
          const u32 jj = b0 + lane;
          p += __popc(__ballot_sync(FULLMASK, jj < q && S.id[jj] < qid));
        }
        if (p == q) continue;
        const u32 vctx = S.ctx[q], vrem = S.rem[q], vinfo = S.info[q], vst = stt[q];
        const i64 vl = S.last[q], vm = S.maxgap[q], va = S.arr[q], vt = S.ttft[q];
        __syncwarp();
        for (u32 c = q; c > p;) {  // shift [p, q) up by one, highest chunk first
          const u32 lo = c > p + 32 ? c - 32 : p;
          const u32 jj = lo + lane;
          const bool v = jj < c;
          u32 a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0;
          i64 b1 = 0, b2 = 0, b3 = 0, b4 = 0;
          if (v) {
            a0 = S.id[jj];
            a1 = S.ctx[jj];
            a2 = S.rem[jj];
            a3 = S.info[jj];
            a4 = stt[jj];
            b1 = S.last[jj];
            b2 = S.maxgap[jj];
            b3 = S.arr[jj];
            b4 = S.ttft[jj];
          }
          __syncwarp();
          if (v) {
            S.id[jj + 1] = a0;
            S.ctx[jj + 1] = a1;
            S.rem[jj + 1] = a2;
            S.info[jj + 1] = a3;
            stt[jj + 1] = a4;
            S.last[jj + 1] = b1;
            S.maxgap[jj + 1] = b2;
            S.arr[jj + 1] = b3;
            S.ttft[jj + 1] = b4;
          }
          __syncwarp();
          c = lo;
        }
        if (lane == 0) {
          S.id[p] = qid;
          S.ctx[p] = vctx;
          S.rem[p] = vrem;
          S.info[p] = vinfo;
          stt[p] = vst;
          S.last[p] = vl;
          S.maxgap[p] = vm;
          S.arr[p] = va;
          S.ttft[p] = vt;
        }
        __syncwarp();
      }
      if (d.nRun == 0) {  // 6. nothing runnable: wake at the next transfer end (or a dispatch)
        d.t = d.xhead_end;
        d.idle = 1;
      } else {
        // 7. cost on the decode profile
        const u32 Dn = d.nRun - nrecomp;
        const u64 Cd = warp_sum64(cdp);
        u64 Np = 0, Ap = 0;
        if (nrecomp) {
          Np = warp_sum64(npp);
          Ap = warp_sum64(app);
        }
        if (KD.preload && swap_in > 0) ev_flush(L);  // the event log doubles as the pipeline's scratch
        const i64 T = iter_time_chunk_ns(KD, Np, Ap, Np, nrecomp, Dn, Cd, swap_out, swap_in,
                                         reinterpret_cast<double *>(L.ev));
        const i64 te = t + T;
        const u64 blocks = totD - d.nfree;
        // 8. commit
        u32 nfin = 0, first_fin = 0xffffffffu, rmin_d = 0xffffffffu;
        const u32 nC = d.nD;  // pulls (now sorted in) may have moved running slots past nA
        #pragma unroll 1
        for (u32 b0 = 0; b0 < nC; b0 += 32) {
          const u32 jj = b0 + lane;
          bool fin = false;
          if (jj < nC) {
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
                             TOKENSIM_REQ_FINISHED, (u32)d.k);
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
            const u32 slot = SLOT(S.info[pos]);
            free_blocks(S.bitmap, btD + (size_t)slot * btl, held, S.id[pos], d.k, koff, L, d.hint);
            d.nfree += held;
            if (lane == 0) atomicOr(&S.btfree[slot >> 5], 1u << (slot & 31u));
          }
        }
        __syncwarp();
        req_iters += d.nRun;
        if (nfin) {
          u32 out = first_fin;
          #pragma unroll 1
          for (u32 b0 = first_fin; b0 < d.nD; b0 += 32) {
            const u32 jj = b0 + lane;
            const bool valid = jj < d.nD;
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
              const u32 dd = out + __popc(km & ltm);
              S.id[dd] = vid;
              S.ctx[dd] = vctx;
              S.rem[dd] = vrem;
              S.info[dd] = vinfo;
              S.last[dd] = vl;
              S.maxgap[dd] = vm;
              S.arr[dd] = va;
              S.ttft[dd] = vt;
              stt[dd] = vst;
            }
            __syncwarp();
            out += __popc(km);
          }
          d.nRun -= nfin;
          d.nD -= nfin;
          done_w += nfin;
          nfin_tot += nfin;
          last_fin = te > last_fin ? te : last_fin;
          tfin_w = t;
        }
        d.rmin = __reduce_min_sync(FULLMASK, rmin_d);
        if (d.nRun == 0) d.rmin = 0;
        fold_iter(d.k, wid, t, T, nrecomp, Dn, Np, Cd, m, nres, nadm, 0, nfin, blocks);
        trace_iter(d.TA, fe, BINNED, FULLT, trcD, P.trace_cap, W, t, te, blocks, flags);
        d.peak = blocks > d.peak ? blocks : d.peak;
        d.bns += blocks * (u64)T;
        swo += swap_out;
        swi += swap_in;
        d.t = te;
        d.last = te;
        ++d.k;
        d.idle = 0;
      }
    }
    return true;
  };
  // one prefill boundary (P_i, i = psel) of the scheduler; false on an internal error
  auto p_step = [&](const u32 psel) -> bool {
    const u32 pi = psel;
    const u32 koff = 2 * pi;
    u32 *bmP = M.bmP + (size_t)pi * P.nwords_max;
    SP.bitmap = bmP;
    u32 *qP = qP0 + (size_t)pi * n;
    u32 *hold = hold0 + (size_t)pi * n;
    u32 *batch = batch0 + (size_t)pi * CAP;
    tokensim_mem_sample *trcP = trc0 + (size_t)pi * P.trace_cap;
    PScal p = M.ps[pi];
    const i64 t = p.t;
    // holders whose transfers ended give their blocks back (any order; ascending list order)
    if (p.hmin <= t) {
      u32 out = 0;
      i64 hm = INF;
      #pragma unroll 1
      for (u32 b0 = 0; b0 < p.nhold; b0 += 32) {
        const u32 x = b0 + lane;
        const bool v = x < p.nhold;
        const u32 id = v ? hold[x] : 0u;
        const i64 xe = v ? reqx[id] : INF;
        const bool fr = v && xe <= t;
        const bool keep = v && !fr;
        hm = (keep && xe < hm) ? xe : hm;
        u32 fm = __ballot_sync(FULLMASK, fr);
        while (fm) {
          const u32 l = (u32)(__ffs(fm) - 1);
          fm &= fm - 1;
          const u32 lid = __shfl_sync(FULLMASK, id, l);
          const u32 ln = B.cdiv(PR[lid]);
          free_blocks(bmP, pblk + (size_t)lid * btl, ln, lid, p.k, koff, L, p.hint);
          p.nfree += ln;
        }
        const u32 km = __ballot_sync(FULLMASK, keep);
        __syncwarp();
        if (keep) hold[out + __popc(km & ltm)] = id;
        __syncwarp();
        out += __popc(km);
      }
#pragma unroll
      for (u32 s = 16; s; s >>= 1) {
        const i64 y = __shfl_xor_sync(FULLMASK, hm, s);
        hm = y < hm ? y : hm;
      }
      p.nhold = out;
      p.hmin = hm;
    }
    // fresh FCFS admission from this worker's dispatch queue into a prefill batch
    u32 nb = 0, E = 0, Kb = 0, nrej = 0;
    u64 tokens = 0, npp = 0, app = 0;
    while (p.qhead < p.qtail) {
      const u32 qi = p.qhead + lane;
      const bool valid = qi < p.qtail;
      const u32 i = valid ? qP[qi] : 0u;
      const u32 pp = valid ? PR[i] : 0u;
      const u32 o = valid ? OU[i] : 0u;
      const u32 need = B.cdiv(pp);
      const bool rej = valid && (u64)need > HPP.cap_fresh;
      const bool el = valid && !rej;
      const u32 ce = scan_incl(el ? 1u : 0u);
      const u32 cneed = scan_incl(el ? need : 0u);
      const u32 cp = scan_incl(el ? pp : 0u);
      const bool ok = el && ((u64)nb + ce <= (u64)mns) && (tokens + cp <= (u64)mbt) &&
                      ((i64)p.nfree - (i64)cneed >= wm);
      const u32 failm = __ballot_sync(FULLMASK, el && !ok);
      const u32 nvalid = min(32u, p.qtail - p.qhead);
      const u32 stop = failm ? (u32)(__ffs(failm) - 1) : nvalid;
      const bool take = el && lane < stop;
      const bool rj = rej && lane < stop;
      const u32 takem = __ballot_sync(FULLMASK, take);
      const u32 cnt = __popc(takem);
      if (take) {
        const u32 rank = __popc(takem & ltm);
        const u32 pos = nb + rank;
        M.pid[pos] = i;
        M.ppl[pos] = pp;
        M.pol[pos] = o;
        M.req_cum[E + rank] = Kb + cneed;
        M.req_pt[E + rank] = pos;
        npp += pp;
        app += (u64)pp * (pp + 1) / 2;
      }
      if (rj) reinterpret_cast<uint8_t *>(rec + i)[26] = (uint8_t)TOKENSIM_REQ_REJECTED;
      const u32 nrj = __popc(__ballot_sync(FULLMASK, rj));
      if (stop) {
        const u32 sneed = __shfl_sync(FULLMASK, cneed, stop - 1);
        const u32 sp = __shfl_sync(FULLMASK, cp, stop - 1);
        p.nfree -= sneed;
        Kb += sneed;
        tokens += sp;
      }
      E += cnt;
      nb += cnt;
      nrej += nrj;
      p.qhead += stop;
      __syncwarp();
      if (stop < nvalid) break;
    }
    nrej_tot += nrej;
    n_done_c += nrej;
    if (nb == 0) {  // idle: wait for a dispatch or for blocks to come back
      p.t = p.hmin;
      p.idle = 1;
    } else {
      if (!alloc_ordered(SP, E, Kb, btP, btl, p.k, koff, L, p.hint, nwP)) {
        flags |= TOKENSIM_PT_INTERNAL_ERROR;
        return false;
      }
      const u64 Np = warp_sum64(npp), Ap = warp_sum64(app);
      const i64 T = iter_time_ns(KP, Np, Ap, nb, 0, 0, 0);
      const i64 te = t + T;
      const u64 blocksP = totP - p.nfree;
      // commit: the first token; o == 1 finishes here, the rest become holders whose block
      // lists move to the per-request table; the whole batch is dispatched onward at te
      u32 nfin = 0;
      #pragma unroll 1
      for (u32 b0 = 0; b0 < nb; b0 += 32) {
        const u32 pos = b0 + lane;
        const bool v = pos < nb;
        const u32 id = v ? M.pid[pos] : 0u, pp = v ? M.ppl[pos] : 0u, o = v ? M.pol[pos] : 0u;
        const bool one = v && o == 1;
        const bool hold_it = v && o > 1;
        const u32 need = B.cdiv(pp);
        if (v) batch[pos] = id;
        if (one) {
          const i64 a = A[id];
          write_record(rec + id, te - a, te - a, 0, 0, TOKENSIM_REQ_FINISHED, (u32)p.k);
        }
        const u32 hm = __ballot_sync(FULLMASK, hold_it);
        if (hold_it) {
          hold[p.nhold + __popc(hm & ltm)] = id;
          reqx[id] = INF;
        }
        u32 vm = __ballot_sync(FULLMASK, v);
        while (vm) {
          const u32 l = (u32)(__ffs(vm) - 1);
          vm &= vm - 1;
          const u32 lpos = b0 + l;
          const u32 lneed = __shfl_sync(FULLMASK, need, l);
          const u32 lid = __shfl_sync(FULLMASK, id, l);
          const bool lone = __shfl_sync(FULLMASK, (u32)one, l) != 0u;
          const u32 *tbl = btP + (size_t)lpos * btl;
          if (lone) {
            free_blocks(bmP, tbl, lneed, lid, p.k, koff, L, p.hint);
            p.nfree += lneed;
          } else {
            #pragma unroll 1
            for (u32 x = lane; x < lneed; x += 32) pblk[(size_t)lid * btl + x] = tbl[x];
          }
        }
        p.nhold += __popc(hm);
        nfin += __popc(__ballot_sync(FULLMASK, one));
        __syncwarp();
      }
      n_done_c += nfin;
      nfin_tot += nfin;
      if (nfin) last_fin = te > last_fin ? te : last_fin;
      fold_iter(p.k, pi, t, T, nb, 0, Np, 0, 0, 0, nb, nrej, nfin, blocksP);
      trace_iter(p.TA, FEp[pi], BINNED, FULLT, trcP, P.trace_cap, W, t, te, blocksP, flags);
      req_iters += nb;
      p.nb = nb;
      p.cur = 0;
      p.tdisp = te;
      p.t = te;
      p.last = te;
      ++p.k;
      p.idle = 0;
    }
    __syncwarp();
    if (lane == 0) M.ps[pi] = p;
    __syncwarp();
    return true;
  };
  // an arrival at ta: dispatched to a prefill worker (no batch completes before the horizon)
  auto arrival_step = [&](const i64 ta) {
    // an arrival: dispatched to a prefill worker (no batch completes before H)
    const u32 pi = pick(false, ta);
    if (lane == 0) {
      PScal &p = M.ps[pi];
      qP0[(size_t)pi * n + p.qtail] = arr;
      p.qtail += 1;
      if (p.idle && ta < p.t) p.t = ta;
    }
    __syncwarp();
    advance_arr();
  };
  // SW, the scheduler warp: fold the decode warps' pull mailboxes into the prefill workers;
  // returns the earliest transfer end folded now
  auto fold_mb = [&]() -> i64 {
    i64 v = INF;
    if (lane < X) {
      v = (i64)atomicExch(reinterpret_cast<unsigned long long *>(&ctl->mb[lane]), (unsigned long long)INF);
      if (v < INF) {
        PScal &p = M.ps[lane];
        if (v < p.hmin) p.hmin = v;
        if (p.idle && v < p.t) p.t = v;
      }
    }
    __syncwarp();
    return min8_i64(v);
  };
  i64 td_next = INF;  // the scheduler warp: the next known end-of-prefill dispatch
  u64 n_epochs = 0, cyc_sched = 0, cyc_dec = 0, cyc_h = 0, cyc_wait = 0;  // profile (point_profile's phase words)
  while (true) {
    // ============================================================ epoch horizon (warp 0)
    const long long c_h0 = clock64();
    if (COORD) {
      u32 nd = n_done_c;
      u32 ef = flags;
      for (u32 w = 0; w < Y; ++w) {
        nd += M.part[w].done;
        ef |= M.part[w].flags;
      }
      i64 H = INF;
      u32 stop = 0;
      if (nd == n || (ef & TOKENSIM_PT_INTERNAL_ERROR)) {
        stop = 1;
      } else {
        const i64 ta = ta_next;
        // tp: the next prefill boundary; tq: the next boundary of a prefill worker with queued
        // requests -- the only boundaries that can start a batch without an arrival first
        i64 tdk = INF, tp = INF, tq = INF, tdm = INF;
        bool blk = false;
        if (lane < X) {
          const PScal &p = M.ps[lane];
          if (p.nb > 0) tdk = p.tdisp;
          tp = p.t;
          blk = p.idle && p.qhead < p.qtail;
          if (p.qhead < p.qtail) tq = p.t;
        }
        if (lane < Y) tdm = M.ds[lane].t;
        tdk = min8_i64(tdk);
        tp = min8_i64(tp);
        tq = min8_i64(tq);
        tdm = min8_i64(tdm);
        const bool blocked = __ballot_sync(FULLMASK, blk) != 0u;
        i64 tall = ta < tdk ? ta : tdk;
        tall = tp < tall ? tp : tall;
        tall = tdm < tall ? tdm : tall;
        if (tall == INF) {
          flags |= TOKENSIM_PT_INTERNAL_ERROR;  // every worker waits: cannot happen under validation
          stop = 1;
        } else if (P.horizon >= 0 && tall >= P.horizon) {
          flags |= TOKENSIM_PT_HORIZON_HIT;
          stop = 1;
        } else {
          H = tdk;
          i64 h1 = sat_add(ta, Tlb);
          // The arrival's own dispatch, exactly: when nothing on the prefill side happens before
          // it (no batch completes, no queued worker's boundary), the arrival is alone at its
          // time and its scheduler choice (round robin / least outstanding: unaffected by the
          // decode phase) is a worker with an empty queue and no batch, whose free blocks admit
          // it now (pulls only return blocks), its batch is {arrival} and dispatches at
          // ta + T(prompt): the decode phase runs to that dispatch, which the scheduler phase
          // then processes -- one epoch per request instead of two.
          if (ta != INF && tdk > ta && tq > ta && P.dispatch != TOKENSIM_DISPATCH_LEAST_MEMORY &&
              ta_next2 != ta) {
            u32 pi;
            if (P.dispatch == TOKENSIM_DISPATCH_ROUND_ROBIN) {
              pi = (u32)(rrP % X);
            } else {
              u64 v = ~0ull;
              if (lane < X) v = (u64)(M.ps[lane].qtail - M.ps[lane].qhead) + M.ps[lane].nb;
              pi = warp_argmin64((i64)v, lane < X);
            }
            const PScal &p = M.ps[pi];
            const u32 pp = pr_next;
            const u32 need = B.cdiv(pp);
            if (p.qhead == p.qtail && p.nb == 0 && (u64)need <= HPP.cap_fresh && mns >= 1u && pp <= mbt &&
                (i64)p.nfree - (i64)need >= wm) {
              const i64 T1 = iter_time_ns(KP, pp, (u64)pp * (pp + 1) / 2, 1, 0, 0, 0);
              h1 = ta + T1;
              const i64 h1n = sat_add(ta_next2, Tlb);  // the next arrival (INF: none)
              h1 = h1n < h1 ? h1n : h1;
            }
          }
          const i64 h2 = sat_add(tq, Tlb);
          H = h1 < H ? h1 : H;
          H = h2 < H ? h2 : H;
          if (blocked) {
            const i64 h3 = sat_add(tdm, Tlb);
            H = h3 < H ? h3 : H;
          }
          if (P.horizon >= 0 && P.horizon < H) H = P.horizon;
        }
      }
      if (lane == 0) {
        ctl->H = H;
        ctl->stop = stop;
      }
    }
    cyc_h += (u64)(clock64() - c_h0);
    __syncthreads();
    if (ctl->stop) break;
    const i64 H = ctl->H;
    const long long c_d0 = clock64();
    if constexpr (SW) {
      // ============ decode warps and the scheduler warp together: every D_j boundary before H,
      // and the scheduler's arrivals and prefill boundaries before H in time order.  A scheduler
      // event at time t waits only for decode warps that could still pull before t (a pull
      // returns prefill blocks at its transfer end): pend = unpulled FIFO entries, prog = the
      // warp's next unprocessed boundary.  Once every remaining request is with the decode
      // workers it waits for all of them, so that it stops at the sequential loop's last event.
      volatile PdnPart *vp = M.part;
      bool c_more = COORD;  // the scheduler warp: events may remain before H
      u32 spins = 0;
      i64 seen_prog = -1;  // lane j < y: decode warp j's last seen progress
      // a wait only fails after ~2^26 polls in which no decode warp advanced (a lost publication)
      auto stalled = [&]() -> bool {
        const i64 pg = lane < Y ? vp[lane].prog : 0;
        if (__any_sync(FULLMASK, pg != seen_prog)) spins = 0;
        seen_prog = pg;
        return ++spins > (1u << 26);
      };
      if (COORD) d.t = INF;
      else d = M.ds[dj];
      auto publish = [&]() {  // lane 0: this decode worker's progress (its data before prog)
        __syncwarp();
        if (lane == 0 && !COORD) {
          vp[dj].done = done_w;
          vp[dj].tfin = tfin_w;
          vp[dj].pend = d.ftail - d.fhead;
          __threadfence_block();
          vp[dj].prog = d.t;
        }
        __syncwarp();
      };
      publish();
      while (true) {
        const i64 tdo = d.t < H ? d.t : INF;
        i64 tc = INF;
        bool c_arr = false;
        u32 psel = 0;
        if (c_more) {
          fold_mb();
          const i64 ta = ta_next;
          const i64 tw = lane < X ? M.ps[lane].t : INF;
          psel = warp_argmin64(tw, lane < X);
          const i64 tb = __shfl_sync(FULLMASK, tw, psel & 31u);
          c_arr = ta <= tb;
          tc = c_arr ? ta : tb;
          if (tc >= H) tc = INF;
        }
        if (tdo <= tc) {
          if (tdo == INF) {
            if (!c_more) break;
            // the scheduler warp, no event before H: a decode warp's pull may still wake a
            // prefill worker, so wait for every decode warp, then look once more
            bool all = true;
            if (lane < Y) all = vp[lane].prog >= H;
            if (__all_sync(FULLMASK, all)) {
              __threadfence_block();
              fold_mb();
              const i64 tw = lane < X ? M.ps[lane].t : INF;
              const i64 tmin = min8_i64(tw);
              if ((ta_next < tmin ? ta_next : tmin) >= H) c_more = false;
              continue;
            }
            __nanosleep(64);
            if (stalled()) {
              flags |= TOKENSIM_PT_INTERNAL_ERROR;
              break;
            }
            continue;
          }
          if (!d_step(H)) break;
          publish();
          continue;
        }
        // a scheduler event at tc (the scheduler warp)
        const bool endgame = n - n_done_c - n_toD == 0u;  // no request before or at a prefill worker
        {
          bool ok = true;
          if (lane < Y) {
            const i64 pg = vp[lane].prog;
            ok = pg > tc || pg >= H || (!endgame && vp[lane].pend == 0u);
          }
          if (!__all_sync(FULLMASK, ok)) {
            __nanosleep(32);
            if (stalled()) {
              flags |= TOKENSIM_PT_INTERNAL_ERROR;
              break;
            }
            continue;
          }
        }
        __threadfence_block();
        if (fold_mb() < tc) continue;  // a pull gave a prefill worker an earlier boundary: re-pick
        if (endgame) {
          // E*: every request is done and no decode worker finished one at or after tc
          u32 ddl = 0;
          i64 tdl = 0;
          if (lane < Y) {
            ddl = vp[lane].done;
            tdl = vp[lane].tfin;
          }
          ddl = __reduce_add_sync(FULLMASK, ddl);
          tdl = -min8_i64(-tdl);
          if (n_done_c + ddl == n && tc >= tdl) {
            c_more = false;
            continue;
          }
        }
        const long long c_e0 = clock64();
        if (c_arr) {
          arrival_step(tc);
        } else if (!p_step(psel)) {
          break;
        }
        cyc_sched += (u64)(clock64() - c_e0);
      }
      __syncwarp();
      if (lane == 0) {
        if (!COORD) M.ds[dj] = d;
        M.part[wib].done = done_w;
        M.part[wib].tfin = tfin_w;
        M.part[wib].flags = flags;
      }
    } else {
      // ============================================ decode phase: every D_j boundary before H
      d = M.ds[dj];
      while (d.t < H)
        if (!d_step(H)) break;
      __syncwarp();
      if (lane == 0) {
        M.ds[dj] = d;
        M.part[dj].done = done_w;
        M.part[dj].tfin = tfin_w;
        M.part[dj].flags = flags;
      }
    }
    const long long c_d1 = clock64();
    cyc_dec += (u64)(c_d1 - c_d0);
    __syncthreads();
    if (!COORD) continue;
    const long long c_s0 = clock64();
    cyc_wait += (u64)(c_s0 - c_d1);
    ++n_epochs;
    if constexpr (SW) fold_mb();  // every pull of the phase (the barrier made them visible)
    // The sequential loop stops at the event that finishes the last request (E*): once every
    // request is done, only events before the decode workers' last finishing boundary (decode
    // boundaries precede prefill boundaries at equal times) are still processed.
    u32 dd = 0;
    i64 tD = 0;
    for (u32 w = 0; w < Y; ++w) {
      dd += M.part[w].done;
      tD = M.part[w].tfin > tD ? M.part[w].tfin : tD;
    }
    // ======================= scheduler phase (warp 0): arrivals and P boundaries before H, in
    // time order (an arrival before a boundary at the same time), then the dispatches at H
    // (SW: the events before H ran alongside the decode warps)
    while (!SW) {
      const i64 ta = ta_next;
      const i64 tw = lane < X ? M.ps[lane].t : INF;
      const u32 psel = warp_argmin64(tw, lane < X);
      const i64 tb = __shfl_sync(FULLMASK, tw, psel & 31u);
      if (ta >= H && tb >= H) break;
      if (n_done_c + dd == n && (ta < tb ? ta : tb) >= tD) break;
      if (ta <= tb) {
        arrival_step(ta);
        continue;
      }
      if (!p_step(psel)) break;
    }
    cyc_sched += (u64)(clock64() - c_s0);
    {  // the next known dispatch, now (a batch started in this phase may end exactly at H)
      const i64 tdl = (lane < X && M.ps[lane].nb > 0) ? M.ps[lane].tdisp : INF;
      td_next = min8_i64(tdl);
      if (td_next < H && n_done_c + dd != n) flags |= TOKENSIM_PT_INTERNAL_ERROR;  // the decode phase ran past it
    }
    if ((flags & TOKENSIM_PT_INTERNAL_ERROR) || td_next != H || (P.horizon >= 0 && H >= P.horizon) ||
        n_done_c + dd == n)
      continue;
    {
      const i64 td = H;
      // ================================================ dispatch events at td, request-id order
      if (lane == 0)
        for (u32 w = 0; w < X; ++w)
          if (M.ps[w].nb > 0 && M.ps[w].tdisp == td) M.ps[w].cur = 0;
      __syncwarp();
      while (true) {
        // the smallest id among completing batches' heads, else an arrival at td
        u32 hid = 0xffffffffu;
        if (lane < X) {
          const PScal &p = M.ps[lane];
          if (p.nb > 0 && p.tdisp == td && p.cur < p.nb) hid = batch0[(size_t)lane * CAP + p.cur];
        }
        const u32 mid = __reduce_min_sync(FULLMASK, hid);
        if (mid != 0xffffffffu) {
          const u32 src = __ffs(__ballot_sync(FULLMASK, hid == mid)) - 1;
          if (lane == 0) M.ps[src].cur += 1;
          __syncwarp();
          if (OU[mid] > 1) {  // o = 1 finished on its prefill worker
            ++n_toD;
            const u32 dq = pick(true, td);
            if (lane == 0) {
              DScal &d = M.ds[dq];
              FifoEnt e;
              e.id = mid;
              e.seg = src;  // the prefill worker holding its blocks
              e.len = B.cdiv(PR[mid]);
              e.pad = 0;
              e.join = td;
              e.xend = INF;
              fifo0[(size_t)dq * n + d.ftail] = e;
              d.ftail += 1;
              if (d.idle && td < d.t) d.t = td;
            }
            __syncwarp();
          }
          continue;
        }
        if (ta_next == td) {
          const u32 pi = pick(false, td);
          if (lane == 0) {
            PScal &p = M.ps[pi];
            qP0[(size_t)pi * n + p.qtail] = arr;
            p.qtail += 1;
            if (p.idle && td < p.t) p.t = td;
          }
          __syncwarp();
          advance_arr();
          continue;
        }
        break;
      }
      if (lane == 0)
        for (u32 w = 0; w < X; ++w)
          if (M.ps[w].nb > 0 && M.ps[w].tdisp == td) {
            M.ps[w].nb = 0;
            M.ps[w].tdisp = INF;
          }
      __syncwarp();

    }
  }
  // ---- termination: every warp hands in its partials; warp 0 flushes traces, writes the
  // records of unfinished requests and the stats
  ev_flush(L);
  pdn_it_flush(L, itcur);
  {
    const u64 dig_s = warp_sum64(L.dig_s);
    const u64 dig_b = warp_sum64(L.dig_b);
    if (lane == 0) {
      PdnPart &q = M.part[wib];
      q.req_iters = req_iters;
      q.npre = npre;
      q.swo = swo;
      q.swi = swi;
      q.nfin = nfin_tot;
      q.n_xfer = n_xfer;
      q.xbytes = xbytes;
      q.ff_iters = ff_iters;
      q.ff_runs = ff_runs;
      q.dig_s = dig_s;
      q.dig_b = dig_b;
      q.last_fin = last_fin;
      q.flags = flags;
      q.done = done_w;
      q.fe = fe;
      q.dcyc = cyc_dec;
    }
  }
  __syncthreads();
  if (COORD) {
    i64 t_final = 0;
    u64 kall = 0, peak = 0, bns = 0;
    for (u32 w = 0; w < NW; ++w) {
      const bool isD = w >= X;
      i64 lw;
      if (isD) {
        const DScal &d = M.ds[w - X];
        lw = d.last;
        kall += d.k;
        peak = d.peak > peak ? d.peak : peak;
        bns += d.bns;
      } else {
        lw = M.ps[w].last;
        kall += M.ps[w].k;
      }
      t_final = lw > t_final ? lw : t_final;
    }
    u64 s_req_iters = 0, s_npre = 0, s_swo = 0, s_swi = 0, s_nfin = 0, s_xfer = 0, s_xbytes = 0, s_ffi = 0,
        s_ffr = 0, s_dig_s = 0, s_dig_b = 0;
    i64 s_last = 0;
    u32 s_flags = 0;
    for (u32 w = 0; w < Y + (SW ? 1u : 0u); ++w) {  // the decode warps (and the SW scheduler warp)
      const PdnPart &q = M.part[w];
      s_req_iters += q.req_iters;
      s_npre += q.npre;
      s_swo += q.swo;
      s_swi += q.swi;
      s_nfin += q.nfin;
      s_xfer += q.n_xfer;
      s_xbytes += q.xbytes;
      s_ffi += q.ff_iters;
      s_ffr += q.ff_runs;
      s_dig_s += q.dig_s;
      s_dig_b += q.dig_b;
      s_last = q.last_fin > s_last ? q.last_fin : s_last;
      s_flags |= q.flags;
    }
    for (u32 w = 0; w < NW; ++w) {
      const bool isD = w >= X;
      TraceAcc ta = isD ? M.ds[w - X].TA : M.ps[w].TA;
      tokensim_mem_sample *tw = trc0 + (size_t)w * P.trace_cap;
      if (BINNED)
        while ((i64)ta.bin * W < t_final) trace_flush_bin(ta, tw, P.trace_cap, W, s_flags);
      __syncwarp();
      if (lane == 0) {
        if (isD) M.ds[w - X].TA = ta;
        else M.ps[w].TA = ta;
      }
      __syncwarp();
    }
    // unfinished: decode slots and pending entries carry their first-token latency, as do the
    // members of an in-flight prefill batch; queued requests have none
    for (u32 w = 0; w < Y; ++w) {
      u32 *sttw;
      const WarpSmem Sw = dview(M, w, CAP, &sttw);
      const DScal &d = M.ds[w];
      #pragma unroll 1
      for (u32 x = lane; x < d.nD; x += 32)
        write_record(rec + Sw.id[x], Sw.ttft[x], 0, 0, Sw.info[x] >> 16, TOKENSIM_REQ_UNFINISHED, 0);
      const FifoEnt *fw = fifo0 + (size_t)w * n;
      #pragma unroll 1
      for (u32 x = d.fhead + lane; x < d.ftail; x += 32) {
        const u32 id = fw[x].id;
        write_record(rec + id, fw[x].join - A[id], 0, 0, 0, TOKENSIM_REQ_UNFINISHED, 0);
      }
    }
    for (u32 w = 0; w < X; ++w) {
      const PScal &p = M.ps[w];
      if (p.nb == 0) continue;
      #pragma unroll 1
      for (u32 x = lane; x < p.nb; x += 32) {
        const u32 id = batch0[(size_t)w * CAP + x];
        if (OU[id] > 1) write_record(rec + id, p.tdisp - A[id], 0, 0, 0, TOKENSIM_REQ_UNFINISHED, 0);
      }
    }
    if (lane == 0) {
      SimStats st;
      st.flags = s_flags | ((nrej_tot == n) ? (u32)TOKENSIM_PT_ALL_REJECTED : 0u);
      st.pad = 0;
      st.n_finished = s_nfin;
      st.n_rejected = nrej_tot;
      st.n_iterations = kall;
      st.n_req_iters = s_req_iters;
      st.n_preempt = s_npre;
      st.swap_out = s_swo;
      st.swap_in = s_swi;
      st.last_finish = s_last;
      st.t_final = t_final;
      st.sched_d = s_dig_s;
      st.block_d = s_dig_b;
      st.req_d = 0;
      st.total_blocks = (u64)Y * totD;  // the decode pool (reading R-X5)
      st.peak_blocks = peak;
      st.block_ns_sum = bns;
      for (u32 w = 0; w < PDN_MAXW; ++w) {
        u64 tn = 0, fn = 0, fb = 0;
        if (w < NW) {
          const TraceAcc &ta = w < X ? M.ps[w].TA : M.ds[w - X].TA;
          const FullEnc &f = w < X ? FEp[w] : M.part[w - X].fe;
          tn = ta.tn;
          fn = f.n;
          fb = f.bytes;
        }
        st.trace_n[w] = FULLT ? fn : (tn < P.trace_cap ? tn : P.trace_cap);
        st.trace_b[w] = fb;
      }
      st.iter_n = kall < P.it_cap ? kall : P.it_cap;
      st.n_transfers = s_xfer;
      st.transfer_bytes = s_xbytes;
      st.ff_iters = s_ffi;
      st.ff_runs = s_ffr;
      st.cycles = (u64)(clock64() - clk0);
      st.cyc_ff = 0;
      st.cyc_ff_fail = 0;
      st.cyc_normal = 0;
      for (int q = 0; q < 8; ++q) st.phase[q] = 0;
      // profile: epochs, scheduler-phase cycles (warp 0), decode-phase cycles of warp 0, the
      // largest and the summed decode-phase cycles over the decode warps
      st.phase[0] = n_epochs;
      st.phase[1] = cyc_sched;
      st.phase[2] = M.part[SW ? Y : 0u].dcyc;  // the scheduler warp's phases
      for (u32 w = 0; w < Y; ++w) {
        st.phase[3] = M.part[w].dcyc > st.phase[3] ? M.part[w].dcyc : st.phase[3];
        st.phase[4] += M.part[w].dcyc;
      }
      st.phase[5] = cyc_h;     // warp 0: horizon computations
      st.phase[6] = cyc_wait;  // warp 0: waiting for the slowest decode warp
      for (int q = 0; q < 8; ++q) st.nphase[q] = 0;
      st.n_req = P.n_req;
      for (int q = 0; q < 5; ++q) st.ff_fail[q] = 0;
      for (int q = 0; q < 5; ++q) st.ff_cut[q] = 0;
      P.stats[j] = st;
    }
  }
  __syncthreads();  // the CTA's next point reuses the shared memory
}

// One CTA per node point: y warps (warp j runs decode worker j; warp 0 also the scheduler and
// the prefill workers), points taken from the LPT queue.  TWO (y <= 6 and more points than
// SMs): registers capped at 168 so two CTAs share an SM.  Measured on c6 (256 points): one
// point alone 208 -> 258 ms (spills), two per SM 1.4x slower each, the sweep 367 ms either way
// (one wave of pairs vs two waves of singles); it pays once the points fill both waves.
// SW (one wave: at most one point per SM): y + 1 warps, the scheduler on a warp of its own that
// runs its events alongside the decode phases (one c6 point alone 190 -> 167 ms).
template <int CAP, bool P2, bool TWO, bool SW>
__global__ void __launch_bounds__(TWO ? 192 : 256, TWO ? 2 : 1) sim_node_kernel(SweepParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ u32 s_qi;
  const u32 wib = threadIdx.x >> 5;
  u32 *bt = P.bt + (size_t)blockIdx.x * P.bt_tables * CAP * P.bt_len;
  while (true) {
    if (threadIdx.x == 0) s_qi = atomicAdd(P.queue, 1u);
    __syncthreads();
    const u32 qi = s_qi;
    __syncthreads();
    if ((u64)qi >= P.n_run) break;
    simulate_pdn<CAP, P2, SW>(P, P.order[qi], smem_raw, bt, wib);
  }
}
