// The fused Q(f2, f3) kernel for sm_100a (included by bfq_cuda.cu).
//
// Q[k1,q1] = sum_tau sum_{a,b} R[k1,a,b,tau] Phi_{tau,q1}[a,b]
// Phi_{tau,q1}[a,b] = sum_{z in slice(tau,q1)} g_z f2[a,q2_z] f3[b,q3_z]
// (the reference's angular-first order, contraction.py:293-317).
//
// CTA = one tile of CELLS cells (staged in shared memory) x up to two teams of
// compute warps.  A team walks the channel list of one l1 group in lockstep
// behind its own R ring (cp.async.bulk + mbarrier; the last warp of the team
// to release a slot refills it).
// Each compute warp owns 8 DMMA rows "pairs" = (m1, cell), M1T = 8/CELLS
// output columns for all CELLS cells, and for every channel runs
//   stage 1  Phi_pair = A B^T over the slice rows: DMMA.8x8x4, M=a, N=b,
//            K=4 table rows per step; the CG-table row (q2, q3, g) of a step is
//            shared by all CELLS cells, operands gathered from the staged f;
//            the row stream is prefetched (next channel's rows into L1, the
//            next k-step's row into registers);
//   stage 2  out[pair,k1] += Phi[pair,(a,b)] R_tau[k1,(a,b)]: DMMA.8x8x4,
//            M=pairs, N=k1, K=n_k^2, two interleaved accumulator sets;
//   epilogue the accumulator of a pair IS Q[cell][k1][q1]: stored once, no
//            atomics, deterministic; exact 0.0 on the invariant slots
//            (kinematic.py:594-610).
//
// Template: MT = ceil(n_k/8) tiles per radial axis, CELLS per tile, BILIN
// (f3 != f2: two staged arrays, no folding), NKT/QST = compile-time n_k and f
// row stride (0 = runtime) so every gather uses an immediate offset.

template <int MT, int CELLS, bool BILIN, int NKT, int QST>
__global__ void __launch_bounds__(256, 1) bfq_q_kernel(const KParams p) {
  constexpr int M1T = 8 / CELLS;
  constexpr bool FIXED = NKT > 0;
  constexpr int NF = BILIN ? 2 : 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = lane >> 2, kq = lane & 3;
  const int NK = FIXED ? NKT : p.nk;
  const int QS = FIXED ? QST : p.qs;
  const int K2P = FIXED ? (NKT * NKT + 3) / 4 * 4 : p.k2p;
  const int K2S = FIXED ? conflict_free_stride_dev((NKT * NKT + 3) / 4 * 4) : p.k2s;
  const int NST = p.nstage;

  long long item_idx, tile;
  cta_item_tile((long long)blockIdx.x, p.n_tiles, p.n_items, p.tile_chunk, item_idx, tile);
  const Item item = p.items[item_idx];

  // shared layout: barriers + arrival counters | R rings (team, stage) | Phi (per warp, 8 pairs) | f (cells)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);  // [team*2 + stage]
  int* arrivals = reinterpret_cast<int*>(full + 8);         // [team*2 + stage]
  int* ctau = arrivals + 8;                                   // [team][max_chan] R block index
  double* rs = reinterpret_cast<double*>(smem_raw + p.hdr);
  const int rblk = NK * K2S;
  double* phis = rs + p.nteams * NST * rblk;  // R rings: nteams x NST slots
  double* fs = phis + p.nw * 8 * K2S;
  const int cell_elems = NK * QS;

  const unsigned rbytes = (unsigned)rblk * 8u;
  // R ring protocol (no producer warp): thread 0 issues the first NST
  // cp.async.bulk loads of each team; afterwards the last warp of a team to
  // finish with a slot (smem arrival counter) issues the refill of that slot.
  auto issue_r = [&](int t, int i, int tau) {
    const int s = i % NST;
    mbar_arrive_expect_tx(&full[t * 2 + s], rbytes);
    bulk_g2s(rs + (t * NST + s) * rblk, p.R + (size_t)tau * rblk, rbytes, &full[t * 2 + s]);
  };
  if (threadIdx.x == 0) {
    for (int t = 0; t < MAX_TEAMS; ++t)
      for (int s = 0; s < NST; ++s) {
        mbar_init(&full[t * 2 + s], 1);
        arrivals[t * 2 + s] = 0;
      }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    for (int t = 0; t < MAX_TEAMS; ++t)
      if (item.nunits[t] > 0) {
        const Group g = p.groups[item.l1[t]];
        for (int i = 0; i < NST && i < g.n_chan; ++i) issue_r(t, i, p.chans[g.chan_off + i].tau);
      }
  }
  // channel R-block indices of both teams, for the refills
  for (int t = 0; t < MAX_TEAMS; ++t)
    if (item.nunits[t] > 0) {
      const Group g = p.groups[item.l1[t]];
      for (int i = threadIdx.x; i < g.n_chan; i += blockDim.x) ctau[t * p.max_chan + i] = p.chans[g.chan_off + i].tau;
    }
  // Phi padding columns (n_k^2 .. k2p) are read by stage 2 and must be 0.
  for (int i = threadIdx.x; i < p.nw * 8 * K2S; i += blockDim.x) phis[i] = 0.0;
  // stage the tile's cells: global (cell, k, q) -> shared (cell, k, q padded to QS);
  // one warp per (array, cell, k) row, lanes over q
  {
    const int rows_total = NF * CELLS * NK;
    const int nwarps = blockDim.x >> 5;
    for (int row = warp; row < rows_total; row += nwarps) {
      const int arr = row / (CELLS * NK);
      const int rem = row - arr * CELLS * NK;
      const int c = rem / NK, k = rem - c * NK;
      const long long cell = tile * CELLS + c;
      const bool ok = cell < p.n_cells;
      const double* src = (arr == 0 ? p.f2 : p.f3) + (ok ? cell : 0) * (long long)NK * p.nq + (long long)k * p.nq;
      double* dst = fs + (arr * CELLS + c) * cell_elems + k * QS;
      for (int q = lane; q < p.nq; q += 32) dst[q] = ok ? __ldg(src + q) : 0.0;
    }
  }
  __syncthreads();

  // team of this unit slot: teams own consecutive slots (scalar selects; a
  // dynamically indexed Item would live in local memory)
  int team = -1, tunit = 0, t_l1 = 0, t_ubase = 0, t_nunits = 0;
  {
    int cum = 0;
#pragma unroll
    for (int t = 0; t < MAX_TEAMS; ++t) {
      const int n = item.nunits[t];
      if (team < 0 && warp < cum + n) {
        team = t;
        tunit = warp - cum;
        t_l1 = item.l1[t];
        t_ubase = item.ubase[t];
        t_nunits = n;
      }
      cum += n;
    }
  }
  if (team < 0) return;
  const int twarp = tunit;
  // ---------------- compute warp
  const bool clk_on = (p.debug & 8) != 0;
  long long ck_s1 = 0, ck_w = 0, ck_s2 = 0, ck_rf = 0, ck0 = clock64(), ckt = ck0;
  const Group grp = p.groups[t_l1];
  const int unit = t_ubase + twarp;
  int m1s[M1T];  // this warp's output columns (plan-balanced), -1 = empty slot
#pragma unroll
  for (int ml = 0; ml < M1T; ++ml) m1s[ml] = p.unit_m1[(grp.unit_off + unit) * M1T + ml];
  uint64_t* tfull = full + team * 2;
  int* tarr = arrivals + team * 2;
  const uint32_t ring_u32 = smem_u32(rs + team * NST * rblk);
  const uint32_t phw_u32 = smem_u32(phis + warp * 8 * K2S);
  const uint32_t cell_bytes = (uint32_t)cell_elems * 8u;
  // Operand rows beyond n_k (DMMA padding) read a clamped valid row: their
  // products only reach accumulator entries (a or b >= n_k, k1 >= n_k) that
  // are never stored, so no zero padding or predication is needed.
  uint32_t fa[MT], fb[MT], rrow[MT];
  {
    const uint32_t f0 = smem_u32(fs);
    const uint32_t f3off = BILIN ? (uint32_t)(CELLS * cell_elems) * 8u : 0u;
#pragma unroll
    for (int t = 0; t < MT; ++t) {
      const int r = min(r0 + 8 * t, NK - 1);
      fa[t] = f0 + (uint32_t)(r * QS) * 8u;
      fb[t] = fa[t] + f3off;
      rrow[t] = (uint32_t)(r * K2S + kq) * 8u;
    }
  }
  double acc2[MT][2], accb[MT][2];
#pragma unroll
  for (int j = 0; j < MT; ++j) acc2[j][0] = acc2[j][1] = accb[j][0] = accb[j][1] = 0.0;

  const int nch = grp.n_chan;
  auto slice_bounds = [&](int ci, int* zs, int* ze) {
    const ChanEntry ce = p.chans[grp.chan_off + ci];
#pragma unroll
    for (int ml = 0; ml < M1T; ++ml) {
      const int m1 = m1s[ml];
      const bool ok = m1 >= 0;
      zs[ml] = ok ? __ldg(p.sstart + ce.slice_base + m1) : 0;
      ze[ml] = ok ? __ldg(p.sstart + ce.slice_base + m1 + 1) : 0;
    }
  };
  auto prefetch_rows_l1 = [&](const int* zs, const int* ze) {
    // 8 rows (128 B) per line, one line per lane
#pragma unroll
    for (int ml = 0; ml < M1T; ++ml)
      for (int z = (zs[ml] & ~7) + lane * 8; z < ze[ml]; z += 256)
        asm volatile("prefetch.global.L1 [%0];\n" ::"l"(p.rows + z));
  };
  // accumulator (a = 8A + r0, b = 8B + 2kq + e) -> Phi row of pair (ml, cc)
  auto store_phi = [&](int ml, double (&acc)[CELLS][MT][MT][2]) {
#pragma unroll
    for (int cc = 0; cc < CELLS; ++cc) {
      const uint32_t ph = phw_u32 + (uint32_t)((ml * CELLS + cc) * K2S) * 8u;
#pragma unroll
      for (int a = 0; a < MT; ++a)
#pragma unroll
        for (int b = 0; b < MT; ++b)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int ia = 8 * a + r0, ib = 8 * b + 2 * kq + e;
            // K in store order (bfq_internal.h phi_k), as the R blocks
            if (ia < NK && ib < NK)
              sts_v(ph + (uint32_t)(phi_base(NK, a, b, e) + r0 * kq_count(NK, b, e) + kq) * 8u, acc[cc][a][b][e]);
          }
    }
  };

  // slice bounds run two channels ahead (their sstart loads come from L2),
  // the L1 row prefetch one channel ahead
  int zs_n[M1T], ze_n[M1T], zs_nn[M1T], ze_nn[M1T];
  slice_bounds(0, zs_n, ze_n);
  if (nch > 1) slice_bounds(1, zs_nn, ze_nn);
  prefetch_rows_l1(zs_n, ze_n);
  Row nxt_row = fetch_row_bf(p.rows, zs_n[0] + kq, ze_n[0]);

  for (int i = 0; i < nch; ++i) {
    int zs[M1T], ze[M1T];
#pragma unroll
    for (int ml = 0; ml < M1T; ++ml) {
      zs[ml] = zs_n[ml];
      ze[ml] = ze_n[ml];
    }
    if (i + 1 < nch) {
#pragma unroll
      for (int ml = 0; ml < M1T; ++ml) {
        zs_n[ml] = zs_nn[ml];
        ze_n[ml] = ze_nn[ml];
      }
      if (i + 2 < nch) slice_bounds(i + 2, zs_nn, ze_nn);
      prefetch_rows_l1(zs_n, ze_n);
    }
    // ---- stage 1: Phi for this warp's 8 (m1, cell) pairs
#pragma unroll
    for (int ml = 0; ml < M1T; ++ml) {
      double acc[CELLS][MT][MT][2];
#pragma unroll
      for (int cc = 0; cc < CELLS; ++cc)
#pragma unroll
        for (int a = 0; a < MT; ++a)
#pragma unroll
          for (int b = 0; b < MT; ++b) acc[cc][a][b][0] = acc[cc][a][b][1] = 0.0;
      const int zend = (p.debug & 1) ? zs[ml] : ze[ml];
      for (int z0 = zs[ml]; z0 < zend; z0 += 4) {
        const Row rw = nxt_row;
        // next row of the stream: this slice, else the next slice, else the
        // first slice of the next channel
        {  // branch-free: select the position, then one unconditional load
          const bool same = z0 + 4 < ze[ml];
          const int zn = ml + 1 < M1T ? zs[ml + 1 < M1T ? ml + 1 : ml] : zs_n[0];
          const int en = ml + 1 < M1T ? ze[ml + 1 < M1T ? ml + 1 : ml] : (i + 1 < nch ? ze_n[0] : 0);
          nxt_row = fetch_row_bf(p.rows, (same ? z0 + 4 : zn) + kq, same ? ze[ml] : en);
        }
        const uint32_t qa = (uint32_t)rw.q2 * 8u, qb = (uint32_t)rw.q3 * 8u;
#pragma unroll
        for (int cc = 0; cc < CELLS; ++cc) {
          double av[MT], bv[MT];
#pragma unroll
          for (int t = 0; t < MT; ++t) {
            av[t] = rw.g * lds_ro(fa[t] + qa + cc * cell_bytes);
            bv[t] = lds_ro(fb[t] + qb + cc * cell_bytes);
          }
#pragma unroll
          for (int a = 0; a < MT; ++a)
#pragma unroll
            for (int b = 0; b < MT; ++b) dmma884(acc[cc][a][b][0], acc[cc][a][b][1], av[a], bv[b]);
        }
      }
      // empty slice: the stream skips it, keep the prefetch pointing at the next one
      if (zs[ml] >= ze[ml]) {
        if (ml + 1 < M1T) nxt_row = fetch_row_bf(p.rows, zs[ml + 1 < M1T ? ml + 1 : ml] + kq, ze[ml + 1 < M1T ? ml + 1 : ml]);
        else nxt_row = fetch_row_bf(p.rows, zs_n[0] + kq, i + 1 < nch ? ze_n[0] : 0);
      }
      if (!(p.debug & 32)) store_phi(ml, acc);
    }
    __syncwarp();
    if (clk_on) { const long long t = clock64(); ck_s1 += t - ckt; ckt = t; }
    // ---- stage 2: out[pair, k1] += Phi[pair, :] . R_tau[k1, :]
    const int s = i % NST;
    mbar_wait_chk(p, &tfull[s], (unsigned)(i / NST) & 1u);
    if (clk_on) { const long long t = clock64(); ck_w += t - ckt; ckt = t; }
    const uint32_t rb = ring_u32 + (uint32_t)(s * rblk) * 8u;
    const uint32_t pa = phw_u32 + (uint32_t)(r0 * K2S + kq) * 8u;
    auto step2 = [&](int k0) {
      const double av0 = lds_v(pa + k0 * 8), av1 = lds_v(pa + (k0 + 4) * 8);
      double bv0[MT], bv1[MT];
#pragma unroll
      for (int j = 0; j < MT; ++j) {
        bv0[j] = lds_v(rb + rrow[j] + k0 * 8);
        bv1[j] = lds_v(rb + rrow[j] + (k0 + 4) * 8);
      }
#pragma unroll
      for (int j = 0; j < MT; ++j) {
        dmma884(acc2[j][0], acc2[j][1], av0, bv0[j]);
        dmma884(accb[j][0], accb[j][1], av1, bv1[j]);
      }
    };
    int k0 = 0;
    if (p.debug & 2) {
      k0 = K2P;
    } else {
      // kept as a loop: a fully unrolled stage 2 lets the compiler sink the
      // next channel's table-row load below it (exposing its L2 latency)
#pragma unroll 2
      for (; k0 + 8 <= K2P; k0 += 8) step2(k0);
    }
    if (k0 < K2P) {  // K2P is a multiple of 4: at most one step left
      const double av = lds_v(pa + k0 * 8);
#pragma unroll
      for (int j = 0; j < MT; ++j) dmma884(acc2[j][0], acc2[j][1], av, lds_v(rb + rrow[j] + k0 * 8));
    }
    __syncwarp();
    if (clk_on) { const long long t = clock64(); ck_s2 += t - ckt; ckt = t; }
    if (lane == 0) {
      // every lane's reads of slot s are complete (consumed by its DMMAs)
      __threadfence_block();
      if (atomicAdd(&tarr[s], 1) == t_nunits - 1) {
        tarr[s] = 0;
        if (i + NST < nch) issue_r(team, i + NST, ctau[team * p.max_chan + i + NST]);
      }
    }
    if (clk_on) { const long long t = clock64(); ck_rf += t - ckt; ckt = t; }
  }
  if (clk_on && lane == 0) {
    atomicAdd(p.dbg_clk + 0, (unsigned long long)ck_s1);
    atomicAdd(p.dbg_clk + 1, (unsigned long long)ck_w);
    atomicAdd(p.dbg_clk + 2, (unsigned long long)ck_s2);
    atomicAdd(p.dbg_clk + 3, (unsigned long long)ck_rf);
    atomicAdd(p.dbg_clk + 4, (unsigned long long)(clock64() - ck0));
    atomicAdd(p.dbg_clk + 5, 1ull);
  }

  // ---------------- epilogue: pair r0 = (m1 = m1s[r0/CELLS], cell = r0%CELLS)
  const int ml = r0 / CELLS, c = r0 - ml * CELLS;
  int m1 = -1;
#pragma unroll
  for (int t = 0; t < M1T; ++t)
    if (t == ml) m1 = m1s[t];
  const long long cell = tile * CELLS + c;
  if (m1 >= 0 && cell < p.n_cells) {
    const int l1 = grp.l1, q1 = l1 * l1 + m1;
#pragma unroll
    for (int j = 0; j < MT; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int k1 = 8 * j + 2 * kq + e;
        if (k1 < NK) {
          double v = acc2[j][e] + accb[j][e];
          if (p.conservation && ((k1 == 0 && l1 <= 1) || (k1 == 1 && l1 == 0))) v = 0.0;
          store_q(p, cell * (long long)NK * p.nq + q1 + (long long)k1 * p.nq, v);
        }
      }
  }
}
