// Pair-split variant of the fused Q(f2, f3) kernel (included by bfq_cuda.cu).
//
// Same algorithm, data layout and plan as bfq_qkernel.cuh, but every unit
// (8 DMMA rows = M1T output columns x CELLS cells) is served by TWO warps:
//   stage 1  warp h of the unit computes Phi for the cells {h*HC .. h*HC+HC-1}
//            (HC = CELLS/2), both warps walk the same table rows (the second
//            read hits L1),
//   stage 2  warp h contracts its half of K = n_k^2 for all 8 pairs; the two
//            partial accumulators are added once, in the epilogue (fixed
//            order, deterministic).
// With 8 units per CTA this gives 16 compute warps (4 per scheduler) in the
// shared memory of 8 (the Phi buffer is per unit), so the 15-cycle issue
// stall of DMMA.8x8x4 and the gather latencies are covered by other warps.
// The two warps of a unit meet at a named barrier twice per channel (Phi
// complete; Phi consumed).

// DUAL (n_k = 17, where shared memory holds only 8 warps): stage 1 walks the
// slice two row groups per iteration into two accumulator sets, doubling the
// independent DMMA chains per warp (ncu at 8 warps: 37% "wait" stalls on the
// single chain); the second group of an odd tail has g = 0 (fetch_row_bf).
template <int MT, int CELLS, bool BILIN, int NKT, int QST>
__global__ void __launch_bounds__(MT == 3 ? (CELLS == 1 ? 384 : 256) : 512, 1) bfq_q_kernel2(const KParams p) {
  constexpr int M1T = 8 / CELLS;
  // Stage-1 split of a unit over its two warps: by cells (warp h takes cells
  // h*HC..h*HC+HC-1, every slice), or -- one cell per tile (SPLITM, n_k = 17:
  // half the staged cells, room for more units) -- by slices (warp h takes
  // slices h*MS..h*MS+MS-1 of the single cell).
  constexpr bool SPLITM = CELLS == 1;
  constexpr int HC = SPLITM ? 1 : CELLS / 2;  // cells per warp in stage 1
  constexpr int MS = SPLITM ? M1T / 2 : M1T;  // slices (output columns m1) per warp in stage 1
  constexpr bool FIXED = NKT > 0;
  constexpr int NF = BILIN ? 2 : 1;
  // 8k+1 sizes (n_k = 9, 17): the last radial index is handled by DFMA +
  // lane reductions instead of a padded DMMA tile row/column (X1); MTM tiles
  // per axis go through DMMA
  constexpr bool X1 = FIXED && (NKT % 8 == 1) && MT >= 2;
  constexpr int MTM = X1 ? MT - 1 : MT;
  // n_k = 9..12 with two cells per warp (MIX): tile (1, 1) of Phi holds at most
  // 4 x 4 useful entries per cell, so the two cells share ONE DMMA -- A rows 0..3
  // from cell 0 (radial rows 8..11), rows 4..7 from cell 1, B columns likewise;
  // the diagonal 4 x 4 blocks of the product are the two cells' tiles, the
  // off-diagonal blocks (cell 0 x cell 1) are dropped.  7 DMMAs per k-step and
  // cell pair instead of 8, for two more gathers.  Same products, same
  // accumulation order, same K numbering: bitwise the unmixed result.
  constexpr bool MIX = FIXED && !X1 && MT == 2 && HC == 2 && NKT > 8 && NKT <= 12;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = lane >> 2, kq = lane & 3;
  const int NK = FIXED ? NKT : p.nk;
  const int QS = FIXED ? QST : p.qs;
  const int K2P = FIXED ? (NKT * NKT + 3) / 4 * 4 : p.k2p;
  const int K2S = FIXED ? conflict_free_stride_dev((NKT * NKT + 3) / 4 * 4) : p.k2s;
  // packed upper triangle of self-symmetric (diag) channels
  const int K2PD = FIXED ? (NKT * (NKT + 1) / 2 + 3) / 4 * 4 : p.k2pd;
  const int K2SD = FIXED ? conflict_free_stride_dev((NKT * (NKT + 1) / 2 + 3) / 4 * 4) : p.k2sd;
  const int NST = p.nstage;
  const int NU = p.nw / 2;  // units (Phi buffers) per CTA

  long long item_idx, tile;
  cta_item_tile((long long)blockIdx.x, p.n_tiles, p.n_items, p.tile_chunk, item_idx, tile);
  const Item item = p.items[item_idx];

  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);  // [team*2 + stage]
  int* arrivals = reinterpret_cast<int*>(full + 8);         // [team*2 + stage]
  int* ctau = arrivals + 8;                                   // [team][max_chan]
  double* rs = reinterpret_cast<double*>(smem_raw + p.hdr);
  const int rblk = NK * K2S;
  double* phis = rs + p.nteams * NST * rblk;  // R rings: nteams x NST slots
  double* fs = phis + NU * 8 * K2S;
  const int cell_elems = NK * QS;

  // ctau[t][i] = 2 * R-block index + diag; diag blocks are shorter (packed K)
  auto issue_r = [&](int t, int i, int code) {
    const int s = NST == 1 ? 0 : (i & 1);
    const unsigned bytes = (unsigned)(NK * ((code & 1) ? K2SD : K2S)) * 8u;
    mbar_arrive_expect_tx(&full[t * 2 + s], bytes);
    bulk_g2s(rs + (t * NST + s) * rblk, p.R + (size_t)(code >> 1) * rblk, bytes, &full[t * 2 + s]);
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
        for (int i = 0; i < NST && i < g.n_chan; ++i) {
          const ChanEntry ce = p.chans[g.chan_off + i];
          issue_r(t, i, 2 * ce.tau + ce.diag);
        }
      }
  }
  for (int t = 0; t < MAX_TEAMS; ++t)
    if (item.nunits[t] > 0) {
      const Group g = p.groups[item.l1[t]];
      for (int i = threadIdx.x; i < g.n_chan; i += blockDim.x) {
        const ChanEntry ce = p.chans[g.chan_off + i];
        ctau[t * p.max_chan + i] = 2 * ce.tau + ce.diag;
      }
    }
  {
    // stage the tile's cells with cp.async (all loads in flight at once; the
    // Phi zeroing below overlaps them); cells past the batch read as zeros
    const int rows_total = NF * CELLS * NK;
    const int nwarps = blockDim.x >> 5;
    for (int row = warp; row < rows_total; row += nwarps) {
      const int arr = row / (CELLS * NK);
      const int rem = row - arr * CELLS * NK;
      const int c = rem / NK, k = rem - c * NK;
      const long long cell = tile * CELLS + c;
      double* dst = fs + (arr * CELLS + c) * cell_elems + k * QS;
      if (cell < p.n_cells) {
        const double* src = (arr == 0 ? p.f2 : p.f3) + cell * (long long)NK * p.nq + (long long)k * p.nq;
        const uint32_t d0 = smem_u32(dst);
        for (int q = lane; q < p.nq; q += 32)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d0 + (uint32_t)q * 8u), "l"(src + q)
                       : "memory");
      } else {
        for (int q = lane; q < p.nq; q += 32) dst[q] = 0.0;
      }
    }
  }
  {
    // Phi rows: every entry a stage-2 k-step can read before the first store
    // overwrites it must be finite -- zero the tail [n_k(n_k+1)/2, K2S) of each
    // row (a packed self-symmetric channel stores only the triangle; the full
    // n_k^2 rows are always written before they are read)
    const int z0 = NK * (NK + 1) / 2, zn = K2S - z0;
    for (int i = threadIdx.x; i < NU * 8 * zn; i += blockDim.x) {
      const int r = i / zn;
      phis[r * K2S + z0 + (i - r * zn)] = 0.0;
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();

  const int u = warp >> 1, h = warp & 1;
  // team of this unit slot: teams own consecutive slots (scalar selects; a
  // dynamically indexed Item would live in local memory)
  int team = -1, tunit = 0, t_l1 = 0, t_ubase = 0, t_nunits = 0;
  {
    int cum = 0;
#pragma unroll
    for (int t = 0; t < MAX_TEAMS; ++t) {
      const int n = item.nunits[t];
      if (team < 0 && u < cum + n) {
        team = t;
        tunit = u - cum;
        t_l1 = item.l1[t];
        t_ubase = item.ubase[t];
        t_nunits = n;
      }
      cum += n;
    }
  }
  if (team < 0) return;  // both warps of an absent unit leave together
  const unsigned bar_id = 1u + (unsigned)u;

#ifdef BFQ_PHASE_CLOCKS
  const bool clk_on = (p.debug & 8) != 0;
  const bool skip1 = (p.debug & 1) != 0, skip2 = (p.debug & 2) != 0;  // timing experiments
  const bool nowait = (p.debug & 4) != 0;  // do not wait for the R ring (stale R: timing only)
  const bool rowhit = (p.debug & 16) != 0;  // fetch table rows 0..15 only (always L1 hits: timing only)
  const bool nostore = (p.debug & 64) != 0;  // skip the per-slice Phi stores (timing only)
  const bool nog = (p.debug & 128) != 0;     // skip the g scaling of the A operand (timing only)
#else
  constexpr bool clk_on = false;  // build with -DBFQ_PHASE_CLOCKS for per-phase cycle counts
  constexpr bool skip1 = false, skip2 = false, nowait = false, rowhit = false, nostore = false, nog = false;
#endif
  long long ck_s1 = 0, ck_b1 = 0, ck_w = 0, ck_s2 = 0, ck_b2 = 0, ck0 = clock64(), ckt = ck0;
  auto tick = [&](long long& acc) {
    if (clk_on) {
      const long long t = clock64();
      acc += t - ckt;
      ckt = t;
    }
  };
  const Group grp = p.groups[t_l1];
  const int unit = t_ubase + tunit;
  const int mlb = SPLITM ? h * MS : 0;  // this warp's first slice of the unit
  const int cb = SPLITM ? 0 : h * HC;    // this warp's first cell of the tile
  int m1s[MS];
#pragma unroll
  for (int ml = 0; ml < MS; ++ml) m1s[ml] = p.unit_m1[(grp.unit_off + unit) * M1T + mlb + ml];
  uint64_t* tfull = full + team * 2;
  int* tarr = arrivals + team * 2;
  const uint32_t ring_u32 = smem_u32(rs + team * NST * rblk);
  const uint32_t phu_u32 = smem_u32(phis + u * 8 * K2S);
  const uint32_t cell_bytes = (uint32_t)cell_elems * 8u;
  uint32_t fa[MT], fb[MT], rrow[MT], rrowd[MT], fx_a = 0, fx_b = 0, rx = 0, rxd = 0;
  uint32_t fa_lo = 0, fb_lo = 0;  // checked builds: this warp's staged cells (f2 / f3)
  const uint32_t fspan = (uint32_t)HC * cell_bytes;
  const uint32_t phu_hi = phu_u32 + (uint32_t)(8 * K2S) * 8u;  // end of this unit's Phi buffer
  {
    const uint32_t f0 = smem_u32(fs) + (uint32_t)cb * cell_bytes;  // this warp's first cell
    const uint32_t f3off = BILIN ? (uint32_t)(CELLS * cell_elems) * 8u : 0u;
#pragma unroll
    for (int t = 0; t < MT; ++t) {
      const int r = min(r0 + 8 * t, NK - 1);
      fa[t] = f0 + (uint32_t)(r * QS) * 8u;
      fb[t] = fa[t] + f3off;
      rrow[t] = (uint32_t)(r * K2S + kq) * 8u;
      rrowd[t] = (uint32_t)(r * K2SD + kq) * 8u;
    }
    if constexpr (MIX) {  // mixed tile: lane row r0 -> cell r0 / 4, radial row 8 + r0 % 4 (clamped)
      fx_a = f0 + (r0 >= 4 ? cell_bytes : 0u) + (uint32_t)(min(8 + (r0 & 3), NK - 1) * QS) * 8u;
    } else
    fx_a = f0 + (uint32_t)((NK - 1) * QS) * 8u;
    fx_b = fx_a + f3off;
    fa_lo = f0;
    fb_lo = f0 + f3off;
    rx = (uint32_t)((NK - 1) * K2S + kq) * 8u;   // R row k1 = n_k-1 (X1 stage 2)
    rxd = (uint32_t)((NK - 1) * K2SD + kq) * 8u;
  }
  double acc2[MT][2], accb[MT][2];
#pragma unroll
  for (int j = 0; j < MT; ++j) acc2[j][0] = acc2[j][1] = accb[j][0] = accb[j][1] = 0.0;
  double x2 = 0.0;  // X1: partial out[pair r0][k1 = n_k-1] over this lane's k

  const int nch = grp.n_chan;
  auto slice_bounds = [&](int ci, int* zs, int* ze) {
    const ChanEntry ce = p.chans[grp.chan_off + ci];
#pragma unroll
    for (int ml = 0; ml < MS; ++ml) {
      const int m1 = m1s[ml];
      const bool ok = m1 >= 0;
      zs[ml] = ok ? __ldg(p.sstart + ce.slice_base + m1) : 0;
      ze[ml] = ok ? __ldg(p.sstart + ce.slice_base + m1 + 1) : 0;
    }
  };
  // Phi is stored in K "store order" (bfq_internal.h phi_k / phid_k): the
  // valid lanes of each half-warp write consecutive doubles, conflict-free.
  // Off-diagonal tiles: base(A,B,e) + r0 * kq_count + kq; diagonal tiles of
  // self-symmetric channels: a per-lane offset computed once here.
  int dpre[MT][2];
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int e = 0; e < 2; ++e)
      dpre[a][e] = phid_base(NK, a, a, e) + diag_rows_before(NK, a, e, r0) - kq_min_diag(r0, e) + kq;
  // MIX: cell 1's tile (1, 1) sits in rows 4..7 x columns 4..7 of the shared accumulator:
  // lane (r0, kq) plays lane (r0 - 4, kq - 2) of an unmixed tile
  const int r0m = r0 & 3, kqm = kq & 1;
  const bool mix_hi = r0 >= 4 && kq >= 2, mix_lo = r0 < 4 && kq < 2;
  int dprem[2];
#pragma unroll
  for (int e = 0; e < 2; ++e)
    dprem[e] = MIX ? phid_base(NK, 1, 1, e) + diag_rows_before(NK, 1, e, r0m) - kq_min_diag(r0m, e) + kqm : 0;
  auto store_phi = [&](int ml, double (&acc)[HC][MT][MT][2], bool dg) {
#pragma unroll
    for (int cc = 0; cc < HC; ++cc) {
      const uint32_t ph = phu_u32 + (uint32_t)(((mlb + ml) * CELLS + cb + cc) * K2S) * 8u;
#pragma unroll
      for (int a = 0; a < MTM; ++a)
#pragma unroll
        for (int b = 0; b < MTM; ++b)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if constexpr (MIX) {
              if (a == 1 && b == 1) {  // shared accumulator acc[0][1][1]
                const int ia = 8 + r0m, ib = 8 + 2 * kqm + e;
                if ((cc == 0 ? mix_lo : mix_hi) && ia < NK && ib < NK && (!dg || ia <= ib)) {
                  const int k = dg ? dprem[e] : phi_base(NK, 1, 1, e) + r0m * kq_count(NK, 1, e) + kqm;
                  sts_v(BFQ_CHK(ph + (uint32_t)k * 8u, ph, ph + (uint32_t)K2S * 8u, CHK_PHI_ST), acc[0][1][1][e]);
                }
                continue;
              }
            }
            const int ia = 8 * a + r0, ib = 8 * b + 2 * kq + e;
            if (!dg) {
              if (ia < NK && ib < NK) {
                const int k = phi_base(NK, a, b, e) + r0 * kq_count(NK, b, e) + kq;
                sts_v(BFQ_CHK(ph + (uint32_t)k * 8u, ph, ph + (uint32_t)K2S * 8u, CHK_PHI_ST), acc[cc][a][b][e]);
              }
            } else if (a <= b && ia <= ib && ib < NK) {
              const int k = a < b ? phid_base(NK, a, b, e) + r0 * kq_count(NK, b, e) + kq : dpre[a][e];
              sts_v(BFQ_CHK(ph + (uint32_t)k * 8u, ph, ph + (uint32_t)K2S * 8u, CHK_PHI_ST), acc[cc][a][b][e]);
            }
          }
    }
  };

  int zs_n[MS], ze_n[MS], zs_nn[MS], ze_nn[MS];
  slice_bounds(0, zs_n, ze_n);
  if (nch > 1) slice_bounds(1, zs_nn, ze_nn);
  // slices are padded to whole k-steps with g = 0 rows (bfq_plan.cpp), and a
  // fetch past the last slice reads a valid row that is never used: no clamp
  auto fetch_rb = [&](int z, int ze) {
    (void)ze;
    return load_row(p.rows, (int)BFQ_CHK_IDX((long long)(rowhit ? (z & 15) : z), p.n_rows, CHK_ROW));
  };
  Row nxt_row = fetch_rb(zs_n[0] + kq, ze_n[0]);
  // DUAL: the second row group of the next iteration, also one iteration ahead
  // (rows of a 600k-row table miss L1; ncu showed long-scoreboard stalls on it)
  constexpr bool DUALK = NKT == 17;
  Row nxt_b = DUALK ? fetch_rb(zs_n[0] + 4 + kq, ze_n[0]) : nxt_row;

  for (int i = 0; i < nch; ++i) {
    int zs[MS], ze[MS];
#pragma unroll
    for (int ml = 0; ml < MS; ++ml) {
      zs[ml] = zs_n[ml];
      ze[ml] = ze_n[ml];
    }
    if (i + 1 < nch) {
#pragma unroll
      for (int ml = 0; ml < MS; ++ml) {
        zs_n[ml] = zs_nn[ml];
        ze_n[ml] = ze_nn[ml];
      }
      if (i + 2 < nch) slice_bounds(i + 2, zs_nn, ze_nn);
    }
    const bool dg = (ctau[team * p.max_chan + i] & 1) != 0;
    auto stage1 = [&](auto dgtag) {
      constexpr bool DGC = decltype(dgtag)::value;
      // ---- stage 1: Phi of this warp's HC cells for its MS columns
#pragma unroll
      for (int ml = 0; ml < MS; ++ml) {
        double acc[HC][MT][MT][2];
        double xr[HC][MTM], xc[HC][MTM], xd[HC];  // X1: row / column / corner of index n_k-1
#pragma unroll
        for (int cc = 0; cc < HC; ++cc) {
#pragma unroll
          for (int a = 0; a < MT; ++a)
#pragma unroll
            for (int b = 0; b < MT; ++b) acc[cc][a][b][0] = acc[cc][a][b][1] = 0.0;
#pragma unroll
          for (int t = 0; t < MTM; ++t) xr[cc][t] = xc[cc][t] = 0.0;
          xd[cc] = 0.0;
        }
        constexpr bool DUAL = NKT == 17;  // also with SPLITM: without it 7.5% slower (r02_ab_xsh_dual.txt)
        double acc2[DUAL ? HC : 1][MT][MT][2];
        if constexpr (DUAL) {
#pragma unroll
          for (int cc = 0; cc < HC; ++cc)
#pragma unroll
            for (int a = 0; a < MT; ++a)
#pragma unroll
              for (int b = 0; b < MT; ++b) acc2[cc][a][b][0] = acc2[cc][a][b][1] = 0.0;
        }
        auto group = [&](const Row& rw, double (&ac)[HC][MT][MT][2], double (&xr_)[HC][MTM], double (&xc_)[HC][MTM],
                         double (&xd_)[HC]) {
          const uint32_t qa = (uint32_t)rw.q2 * 8u, qb = (uint32_t)rw.q3 * 8u;
#pragma unroll
          for (int cc = 0; cc < HC; ++cc) {
            double av[MT], bv[MT];
#pragma unroll
            for (int t = 0; t < MTM; ++t) {
              const double fv = lds_ro(BFQ_CHK(fa[t] + qa + cc * cell_bytes, fa_lo, fa_lo + fspan, CHK_F2));
              av[t] = nog ? fv : rw.g * fv;
              bv[t] = lds_ro(BFQ_CHK(fb[t] + qb + cc * cell_bytes, fb_lo, fb_lo + fspan, CHK_F3));
            }
#pragma unroll
            for (int a = 0; a < MTM; ++a)
#pragma unroll
              for (int b = 0; b < MTM; ++b)
                if ((b >= a || !DGC) && !(MIX && a == 1 && b == 1))
                  dmma884(ac[cc][a][b][0], ac[cc][a][b][1], av[a], bv[b]);
            if constexpr (X1) {
              // g f2[n_k-1, q2], f3[n_k-1, q3] of this lane's row kq, cell cc (broadcast
              // loads; one gather + shuffles measured 3.5% slower, profiles/r02_ab_xsh_dual.txt)
              const double ea = rw.g * lds_ro(BFQ_CHK(fx_a + qa + cc * cell_bytes, fa_lo, fa_lo + fspan, CHK_F2));
              const double eb = lds_ro(BFQ_CHK(fx_b + qb + cc * cell_bytes, fb_lo, fb_lo + fspan, CHK_F3));
#pragma unroll
              for (int t = 0; t < MTM; ++t) {
                if (!DGC) xr_[cc][t] = fma(ea, bv[t], xr_[cc][t]);
                xc_[cc][t] = fma(av[t], eb, xc_[cc][t]);
              }
              xd_[cc] = fma(ea, eb, xd_[cc]);
            }
          }
          if constexpr (MIX) {  // tile (1, 1) of both cells in one DMMA
            const double am = rw.g * lds_ro(BFQ_CHK(fx_a + qa, fa_lo, fa_lo + fspan, CHK_F2));
            const double bm = lds_ro(BFQ_CHK(fx_b + qb, fb_lo, fb_lo + fspan, CHK_F3));
            dmma884(ac[0][1][1][0], ac[0][1][1][1], am, bm);
          }
        };
        const int zn = ml + 1 < MS ? zs[ml + 1 < MS ? ml + 1 : ml] : zs_n[0];
        const int en = ml + 1 < MS ? ze[ml + 1 < MS ? ml + 1 : ml] : (i + 1 < nch ? ze_n[0] : 0);
        if constexpr (DUAL) {
          for (int z0 = zs[ml]; z0 < (skip1 ? zs[ml] : ze[ml]); z0 += 8) {
            const Row rwa = nxt_row;
            const Row rwb = nxt_b;  // g = 0 past the slice end
            const bool same = z0 + 8 < ze[ml];
            nxt_row = fetch_rb((same ? z0 + 8 : zn) + kq, same ? ze[ml] : en);
            nxt_b = fetch_rb((same ? z0 + 12 : zn + 4) + kq, same ? ze[ml] : en);
            group(rwa, acc, xr, xc, xd);
            group(rwb, acc2, xr, xc, xd);  // shared X1 sums (separate ones: 3% slower, r02_ab_xsh_dual.txt)
          }
#pragma unroll
          for (int cc = 0; cc < HC; ++cc)
#pragma unroll
            for (int a = 0; a < MT; ++a)
#pragma unroll
              for (int b = 0; b < MT; ++b) {
                acc[cc][a][b][0] += acc2[cc][a][b][0];
                acc[cc][a][b][1] += acc2[cc][a][b][1];
              }
        } else {
          for (int z0 = zs[ml]; z0 < (skip1 ? zs[ml] : ze[ml]); z0 += 4) {
            const Row rw = nxt_row;
            const bool same = z0 + 4 < ze[ml];
            nxt_row = fetch_rb((same ? z0 + 4 : zn) + kq, same ? ze[ml] : en);
            group(rw, acc, xr, xc, xd);
          }
        }
        if (zs[ml] >= ze[ml]) {
          if (ml + 1 < MS) nxt_row = fetch_rb(zs[ml + 1 < MS ? ml + 1 : ml] + kq, ze[ml + 1 < MS ? ml + 1 : ml]);
          else nxt_row = fetch_rb(zs_n[0] + kq, i + 1 < nch ? ze_n[0] : 0);
          if constexpr (DUALK) {
            if (ml + 1 < MS) nxt_b = fetch_rb(zs[ml + 1 < MS ? ml + 1 : ml] + 4 + kq, ze[ml + 1 < MS ? ml + 1 : ml]);
            else nxt_b = fetch_rb(zs_n[0] + 4 + kq, i + 1 < nch ? ze_n[0] : 0);
          }
        }
        if (!nostore) store_phi(ml, acc, DGC);
        if constexpr (X1) {
          // lanes kq = 0..3 hold partial sums over their own rows: reduce, then
          // the kq == 0 lanes store row / column n_k-1 of Phi
#pragma unroll
          for (int cc = 0; cc < HC; ++cc) {
#pragma unroll
            for (int t = 0; t < MTM; ++t) {
              xr[cc][t] += __shfl_xor_sync(0xffffffffu, xr[cc][t], 1);
              xr[cc][t] += __shfl_xor_sync(0xffffffffu, xr[cc][t], 2);
              xc[cc][t] += __shfl_xor_sync(0xffffffffu, xc[cc][t], 1);
              xc[cc][t] += __shfl_xor_sync(0xffffffffu, xc[cc][t], 2);
            }
            xd[cc] += __shfl_xor_sync(0xffffffffu, xd[cc], 1);
            xd[cc] += __shfl_xor_sync(0xffffffffu, xd[cc], 2);
            const uint32_t ph = phu_u32 + (uint32_t)(((mlb + ml) * CELLS + cb + cc) * K2S) * 8u;
            // store-order K of row / column L = n_k - 1 = 8 (MT - 1): tile row or
            // column MT - 1 holds one index (r0 = 0 or kq = e = 0)
            constexpr int L = NKT - 1, TL = MT - 1;
            // after the butterfly every kq lane of row r0 holds the sums: at n_k = 9
            // (shared-memory-bound) lanes kq = 0 store the row value and lanes kq = 1
            // the column value in ONE store per t (2 wavefronts for 16 values;
            // +1.4% there, -0.2% at n_k = 17: profiles/r02_x1_store_ab.txt)
            constexpr bool XCOMB = NKT == 9;
            if (XCOMB ? kq <= 1 : kq == 0) {
#pragma unroll
              for (int t = 0; t < MTM; ++t) {
                if (!DGC) {
                  // Phi[L][8t + r0]: tile (TL, t), half r0 & 1, kq' = r0 >> 1
                  const int kr = ((r0 & 1) ? phi_base(NKT, TL, t, 1) : phi_base(NKT, TL, t, 0)) + (r0 >> 1);
                  // Phi[8t + r0][L]: tile (t, TL), half 0, kq' = 0 (one valid kq)
                  const int kc = phi_base(NKT, t, TL, 0) + r0 * kq_count(NKT, TL, 0);
                  if constexpr (XCOMB) {
                    sts_v(BFQ_CHK(ph + (uint32_t)(kq == 0 ? kr : kc) * 8u, ph, ph + (uint32_t)K2S * 8u, CHK_PHI_ST),
                          kq == 0 ? xr[cc][t] : xc[cc][t]);
                  } else {
                    sts_v(BFQ_CHK(ph + (uint32_t)kr * 8u, ph, ph + (uint32_t)K2S * 8u, CHK_PHI_ST), xr[cc][t]);
                    sts_v(BFQ_CHK(ph + (uint32_t)kc * 8u, ph, ph + (uint32_t)K2S * 8u, CHK_PHI_ST), xc[cc][t]);
                  }
                } else if (kq == 0) {
                  const int kc = phid_base(NKT, t, TL, 0) + r0 * kq_count(NKT, TL, 0);
                  sts_v(BFQ_CHK(ph + (uint32_t)kc * 8u, ph, ph + (uint32_t)K2S * 8u, CHK_PHI_ST), xc[cc][t]);
                }
              }
              if (r0 == 0 && kq == 0) {
                const int pl = DGC ? phid_k(NKT, L, L) : phi_k(NKT, L, L);
                sts_v(BFQ_CHK(ph + (uint32_t)pl * 8u, ph, ph + (uint32_t)K2S * 8u, CHK_PHI_ST), xd[cc]);
              }
            }
          }
        }
      }
    };
    if (dg) stage1(std::true_type{});
    else stage1(std::false_type{});
    tick(ck_s1);
    BFQ_JITTER(4 * i + 1);
    named_bar_sync(bar_id, 64);  // Phi of all 8 pairs written
    tick(ck_b1);
    // ---- stage 2: this warp's half of K for all 8 pairs
    // ring slot and phase of channel i (NST is 1 or 2: no integer division)
    const int s = NST == 1 ? 0 : (i & 1);
    const unsigned par = NST == 1 ? (unsigned)(i & 1) : (unsigned)((i >> 1) & 1);
    BFQ_JITTER(4 * i + 2);
    if (!nowait || i == 0) mbar_wait_chk(p, &tfull[s], par);
    tick(ck_w);
    const uint32_t rb = ring_u32 + (uint32_t)(s * rblk) * 8u;
    const uint32_t rb_hi = rb + (uint32_t)rblk * 8u;  // end of this ring slot
    (void)rb_hi;
    const uint32_t pa = phu_u32 + (uint32_t)(r0 * K2S + kq) * 8u;
    auto stage2 = [&](auto dgtag) {
      constexpr bool DGC = decltype(dgtag)::value;
      // this warp's half of the k-steps (K = n_k^2, or the packed triangle)
      const int nks = (DGC ? K2PD : K2P) / 4;
      const int ks0 = h ? (nks + 1) / 2 : 0, ks1 = skip2 ? ks0 : (h ? nks : (nks + 1) / 2);
      uint32_t rr[MT];
#pragma unroll
      for (int j = 0; j < MT; ++j) rr[j] = DGC ? rrowd[j] : rrow[j];
      const uint32_t rrx = DGC ? rxd : rx;  // X1: R row k1 = n_k-1 (DFMA)
      int ks = ks0;
#pragma unroll 2
      for (; ks + 2 <= ks1; ks += 2) {
        const int k0 = ks * 4;
        const double av0 = lds_v(BFQ_CHK(pa + k0 * 8, phu_u32, phu_hi, CHK_PHI_LD));
        const double av1 = lds_v(BFQ_CHK(pa + (k0 + 4) * 8, phu_u32, phu_hi, CHK_PHI_LD));
        double bv0[MT], bv1[MT];
#pragma unroll
        for (int j = 0; j < MTM; ++j) {
          bv0[j] = lds_v(BFQ_CHK(rb + rr[j] + k0 * 8, rb, rb_hi, CHK_RING));
          bv1[j] = lds_v(BFQ_CHK(rb + rr[j] + (k0 + 4) * 8, rb, rb_hi, CHK_RING));
        }
#pragma unroll
        for (int j = 0; j < MTM; ++j) {
          dmma884(acc2[j][0], acc2[j][1], av0, bv0[j]);
          dmma884(accb[j][0], accb[j][1], av1, bv1[j]);
        }
        if constexpr (X1) {
          x2 = fma(av0, lds_v(BFQ_CHK(rb + rrx + k0 * 8, rb, rb_hi, CHK_RING)), x2);
          x2 = fma(av1, lds_v(BFQ_CHK(rb + rrx + (k0 + 4) * 8, rb, rb_hi, CHK_RING)), x2);
        }
      }
      if (ks < ks1) {
        const int k0 = ks * 4;
        const double av = lds_v(BFQ_CHK(pa + k0 * 8, phu_u32, phu_hi, CHK_PHI_LD));
#pragma unroll
        for (int j = 0; j < MTM; ++j)
          dmma884(acc2[j][0], acc2[j][1], av, lds_v(BFQ_CHK(rb + rr[j] + k0 * 8, rb, rb_hi, CHK_RING)));
        if constexpr (X1) x2 = fma(av, lds_v(BFQ_CHK(rb + rrx + k0 * 8, rb, rb_hi, CHK_RING)), x2);
      }
    };
    if (dg) stage2(std::true_type{});
    else stage2(std::false_type{});
    tick(ck_s2);
    BFQ_JITTER(4 * i + 3);
    named_bar_sync(bar_id, 64);  // Phi consumed by both warps
    tick(ck_b2);
    if constexpr (kChecked) {
      // Race canaries: this warp's Phi rows are poisoned with 1e300 until its
      // next stage 1 rewrites them (a stage-2 read of a stale or early Phi
      // entry blows Q up), and the last warp to release an R slot poisons it
      // before the refill (a read of a released or not-yet-landed slot does
      // the same).  Unused K padding keeps its zeros, so a correct schedule
      // is unaffected: 1e300 x 0 = 0.
#pragma unroll 1
      for (int ml = 0; ml < (i + 1 < nch ? MS : 0); ++ml)  // not after the last channel: the
#pragma unroll 1                                           // epilogue reuses the buffer
        for (int cc = 0; cc < HC; ++cc) {
          const uint32_t ph = phu_u32 + (uint32_t)(((mlb + ml) * CELLS + cb + cc) * K2S) * 8u;
          for (int e = lane; e < NK * NK; e += 32) sts_v(ph + (uint32_t)e * 8u, 1e300);
        }
      __syncwarp();
      BFQ_JITTER(4 * i);
      int last = 0;
      if (lane == 0) {
        __threadfence_block();
        last = atomicAdd(&tarr[s], 1) == 2 * t_nunits - 1;
        if (last) tarr[s] = 0;
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        for (int e = lane; e < NK * K2S; e += 32) sts_v(rb + (uint32_t)e * 8u, 1e300);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0 && i + NST < nch) issue_r(team, i + NST, ctau[team * p.max_chan + i + NST]);
      }
    } else if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&tarr[s], 1) == 2 * t_nunits - 1) {
        tarr[s] = 0;
        if (i + NST < nch) issue_r(team, i + NST, ctau[team * p.max_chan + i + NST]);
      }
    }
  }

  if (clk_on && lane == 0) {
    atomicAdd(p.dbg_clk + 0, (unsigned long long)ck_s1);
    atomicAdd(p.dbg_clk + 1, (unsigned long long)ck_b1);
    atomicAdd(p.dbg_clk + 2, (unsigned long long)ck_w);
    atomicAdd(p.dbg_clk + 3, (unsigned long long)ck_s2);
    atomicAdd(p.dbg_clk + 4, (unsigned long long)ck_b2);
    atomicAdd(p.dbg_clk + 5, (unsigned long long)(clock64() - ck0));
    atomicAdd(p.dbg_clk + 6, 1ull);
  }
  // ---------------- epilogue: warp 1 hands its K-half partials to warp 0
  if constexpr (X1) {  // out[pair][n_k-1]: sum the four kq lanes
    x2 += __shfl_xor_sync(0xffffffffu, x2, 1);
    x2 += __shfl_xor_sync(0xffffffffu, x2, 2);
  }
  const uint32_t xch = phu_u32 + (uint32_t)(lane * (2 * MT + 1)) * 8u;
  if (h == 1) {
#pragma unroll
    for (int j = 0; j < MTM; ++j) {
      sts_v(BFQ_CHK(xch + (uint32_t)(2 * j) * 8u, phu_u32, phu_hi, CHK_XCH), acc2[j][0] + accb[j][0]);
      sts_v(BFQ_CHK(xch + (uint32_t)(2 * j + 1) * 8u, phu_u32, phu_hi, CHK_XCH), acc2[j][1] + accb[j][1]);
    }
    if constexpr (X1) sts_v(BFQ_CHK(xch + (uint32_t)(2 * MT) * 8u, phu_u32, phu_hi, CHK_XCH), x2);
  }
  named_bar_sync(bar_id, 64);
  if (h == 1) return;
  const int ml = r0 / CELLS, c = r0 - ml * CELLS;
  int m1 = -1;
  if constexpr (SPLITM) {
    m1 = p.unit_m1[(grp.unit_off + unit) * M1T + ml];  // all M1T slices (warp 0 staged only its own)
  } else {
#pragma unroll
    for (int t = 0; t < M1T; ++t)
      if (t == ml) m1 = m1s[t];
  }
  const long long cell = tile * CELLS + c;
  if (m1 >= 0 && cell < p.n_cells) {
    const int l1 = grp.l1, q1 = l1 * l1 + m1;
    auto put = [&](int k1, double v) {
      if (p.conservation && ((k1 == 0 && l1 <= 1) || (k1 == 1 && l1 == 0))) {
        // the zeroed R rows (kinematic.py:594-610) already make these sums exactly 0
        if (kChecked && v != 0.0) BFQ_CHK_IDX(1LL, 0LL, CHK_ZERO);
        v = 0.0;
      }
      const long long off = cell * (long long)NK * p.nq + q1 + (long long)k1 * p.nq;
      store_q(p, BFQ_CHK_IDX(off, p.n_cells * (long long)NK * p.nq, CHK_Q), v);
    };
#pragma unroll
    for (int j = 0; j < MTM; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int k1 = 8 * j + 2 * kq + e;
        if (k1 < NK)
          put(k1, (acc2[j][e] + accb[j][e]) +
                      lds_v(BFQ_CHK(xch + (uint32_t)(2 * j + e) * 8u, phu_u32, phu_hi, CHK_XCH)));
      }
    if constexpr (X1)
      if (kq == 0) put(NK - 1, x2 + lds_v(BFQ_CHK(xch + (uint32_t)(2 * MT) * 8u, phu_u32, phu_hi, CHK_XCH)));
  }
}
