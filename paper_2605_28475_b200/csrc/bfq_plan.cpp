// Host-side plan construction for the Q(f,f) engine: operator validation,
// slot-symmetry folding, device data layout, kernel configuration and the
// per-tile CTA schedule.  Pure C++ (no CUDA); bfq_cuda.cu uploads the result.
//
// Reference semantics followed here:
//   * operator validation        -- FactorizedOperator.__post_init__, contraction.py:86-108
//   * (tau, q1) sort guard        -- q_angular_first, contraction.py:297-301
//   * slices over (tau, q1)       -- angular.py:272-285, cache.py:147-150
//   * R layout (n_k,n_k,n_k,N_T)  -- kinematic.py:574-578, cache.py:61,139
//   * BFCT file format            -- cache.py:1-19, :41, :52-63, :92-166
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <unordered_map>

#include "bfq_internal.h"

namespace bfq {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
const std::string& get_error() { return g_err; }

static int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

static inline int isqrt_floor(int x) {
  int r = (int)std::sqrt((double)x);
  while (r * r > x) --r;
  while ((r + 1) * (r + 1) <= x) ++r;
  return r;
}

static int conflict_free_stride(int n) { return conflict_free_stride_dev(n); }

// Shared memory of one CTA: two R rings (one per team) | Phi per warp | f of the tile.
static long smem_bytes(int nk, int qs, int k2s, int nf, int cells, int units, int nstage, int hdr, int nteams) {
  return hdr + (long)nteams * nstage * nk * k2s * 8 + (long)units * 8 * k2s * 8 + (long)nf * cells * nk * qs * 8;
}

// Header region: 8 mbarriers, 8 arrival counters, then the R-block index of
// every channel of both teams (the refill path reads it from shared memory).
static int header_bytes(int max_chan) { return 96 + (MAX_TEAMS * max_chan * 4 + 31) / 32 * 32; }

// DMMA.8x8x4 issues with a ~15-cycle stall on its warp, so a scheduler needs
// at least two compute warps to keep the FP64 tensor pipe fed while the other
// warp issues gathers: prefer 8 compute warps, then fewer cells per tile.
static bool choose_config(int nk, int qs, int k2s, int nf, int smem_limit, int max_chan, KernelConfig& c) {
  c.mt = (nk + 7) / 8;
  c.nf = nf;
  // stage-1 accumulators in registers; n_k = 9 runs its last index on DFMA (X1,
  // bfq_qkernel2.cuh), leaving one 8x8 tile per cell, so it takes 8 cells per tile
  int max_cells = c.mt == 1 ? 8 : (c.mt == 2 ? 4 : 2);
  if (nk == 9 && qs == 84 && !std::getenv("BFQ_GENERIC") && !std::getenv("BFQ_NO_X1_CELLS8")) max_cells = 8;
  int force_cells = 0, kernel = 2;
  if (const char* e = std::getenv("BFQ_CELLS")) force_cells = std::atoi(e);
  if (const char* e = std::getenv("BFQ_KERNEL")) kernel = std::atoi(e);
  c.hdr = header_bytes(max_chan);
  c.max_chan = max_chan;
  // Pair-split kernel first: 8 units x 2 warps (4 compute warps per
  // scheduler) in the shared memory of 8 Phi buffers.  R rings: up to 4 teams
  // with one stage each (measured as fast as two stages: the refill has a
  // whole stage 1 to land), else 2 teams.
  static const int popts[][4] = {  // cells, units, stages, teams
      {8, 8, 1, 4}, {8, 8, 2, 2}, {4, 8, 1, 4}, {4, 8, 1, 3}, {4, 8, 2, 2}, {4, 8, 1, 2},
      {2, 8, 1, 4}, {2, 8, 2, 2}, {2, 8, 1, 2}, {8, 4, 1, 4}, {8, 4, 1, 2}, {4, 4, 1, 4}, {4, 4, 1, 2},
      {2, 4, 1, 4}, {2, 4, 1, 2}, {2, 4, 1, 1}};
  int force_stages = 0, force_teams = 0, force_units = 0;
  if (const char* e = std::getenv("BFQ_STAGES")) force_stages = std::atoi(e);
  if (const char* e = std::getenv("BFQ_TEAMS")) force_teams = std::atoi(e);
  if (const char* e = std::getenv("BFQ_UNITS")) force_units = std::atoi(e);
  // Two CTAs per SM (4 units x 2 warps each, <= 128 registers) when their
  // shared memory fits twice per SM: a CTA's prologue and tail then overlap
  // the other CTA's work (measured +2.6% at N=L=8 and N=L=10).
  static const int popts2[][4] = {{8, 4, 1, 4}, {8, 4, 1, 3}, {8, 4, 1, 2}, {4, 4, 1, 4}, {4, 4, 1, 3}, {4, 4, 1, 2}};
  const long half_sm = (233472L - 2 * 1024) / 2;  // 228 KB per SM, 1 KB reserved per CTA
  if (kernel == 2 && !force_stages && (!force_units || force_units == 4) && nk != 17 &&
      !std::getenv("BFQ_ONE_CTA")) {
    for (auto o0 : popts2) {
      int o[4] = {o0[0], o0[1], o0[2], force_teams ? force_teams : o0[3]};
      if (force_cells && o[0] != force_cells) continue;
      if (o[0] > max_cells || o[3] > MAX_TEAMS) continue;
      const long smem = smem_bytes(nk, qs, k2s, nf, o[0], o[1], o[2], c.hdr, o[3]);
      if (smem > std::min<long>(half_sm, smem_limit)) continue;
      c.cells = o[0];
      c.m1t = 8 / o[0];
      c.upc = o[1];
      c.nw = 2 * o[1];
      c.nstage = o[2];
      c.nteams = o[3];
      c.smem = (int)smem;
      c.cg = c.cells;
      c.pairsplit = 1;
      return true;
    }
  }
  // One cell per tile, the unit's 8 output columns split over its two warps
  // (SPLITM, bfq_qkernel2.cuh): half the staged cells of the 2-cell tile,
  // which at n_k = 17 leaves room for a second R ring or more units.
  // Measured at N=L=16 (16,384 cells): 2 cells x 4 units, 1 ring 42.4k cells/s;
  // 1 cell x 4 units, 2 rings 44.1k; 1 cell x 5 units (10 warps), 2 rings 44.9k;
  // 6 units with 1 ring 36.8k (one l1 group per CTA: packing 0.47).
  // 6 units (12 warps) with 2 rings fill shared memory to 232,288 of 232,448
  // bytes at the folded program's 57 channels per group; registers are
  // allocated per scheduler partition, so 12 warps (3 per partition) have the
  // same 168-register cap as 10: 46.9k -> 51.1k cells/s (profiles/r02_n16_units.txt).
  static const int popts1[][4] = {{1, 6, 1, 2}, {1, 5, 1, 2}, {1, 4, 1, 2}, {1, 6, 1, 1}, {1, 4, 1, 1}};
  // (SPLITM is instantiated for the compile-time n_k = 17 kernel only)
  if (kernel == 2 && nk == 17 && !std::getenv("BFQ_GENERIC") && (force_cells == 1 || !force_cells)) {
    for (auto o0 : popts1) {
      int o[4] = {o0[0], o0[1], o0[2], force_teams ? force_teams : o0[3]};
      if (force_units && o[1] != force_units) continue;
      if (o[3] > MAX_TEAMS) continue;
      const long smem = smem_bytes(nk, qs, k2s, nf, o[0], o[1], o[2], c.hdr, o[3]);
      if (smem > smem_limit) continue;
      c.cells = 1;
      c.m1t = 8;
      c.upc = o[1];
      c.nw = 2 * o[1];
      c.nstage = o[2];
      c.nteams = o[3];
      c.smem = (int)smem;
      c.cg = 1;
      c.pairsplit = 1;
      return true;
    }
  }
  if (kernel == 2) {
    for (auto o0 : popts) {
      int o[4] = {o0[0], o0[1], force_stages ? force_stages : o0[2], force_teams ? force_teams : o0[3]};
      if (force_cells && o[0] != force_cells) continue;
      if (force_units && o[1] != force_units) continue;
      if (o[0] > max_cells || o[0] < 2) continue;
      if (o[2] * o[3] > 2 * MAX_TEAMS || o[3] > MAX_TEAMS || o[2] > 2) continue;
      const long smem = smem_bytes(nk, qs, k2s, nf, o[0], o[1], o[2], c.hdr, o[3]);
      if (smem > smem_limit) continue;
      c.cells = o[0];
      c.m1t = 8 / o[0];
      c.upc = o[1];
      c.nw = 2 * o[1];
      c.nstage = o[2];
      c.nteams = o[3];
      c.smem = (int)smem;
      c.cg = c.cells;
      c.pairsplit = 1;
      return true;
    }
  }
  // Single-warp-per-unit kernel (bfq_qkernel.cuh): only when no pair-split
  // shape fits (e.g. the bilinear Q(f2,f3) program at n_k = 17, whose two
  // staged arrays leave no room for two cells), or forced by BFQ_KERNEL=1.
  static const int opts[][3] = {  // cells, compute warps (= units), ring stages
      {8, 8, 2}, {4, 8, 2}, {4, 8, 1}, {2, 8, 2}, {2, 8, 1}, {8, 4, 2}, {4, 4, 2}, {4, 4, 1},
      {2, 4, 2}, {2, 4, 1}, {1, 8, 1}, {1, 4, 1}, {1, 2, 1}, {1, 1, 1}};
  const int max_cells1 = c.mt == 1 ? 8 : (c.mt == 2 ? 4 : 2);  // no X1 variant of this kernel
  for (auto& o : opts) {
    if (force_cells && o[0] != force_cells) continue;
    if (o[0] > max_cells1) continue;
    const long smem = smem_bytes(nk, qs, k2s, nf, o[0], o[1], o[2], c.hdr, 2);
    if (smem > smem_limit) continue;
    c.cells = o[0];
    c.m1t = 8 / o[0];
    c.nw = o[1];
    c.upc = o[1];
    c.nteams = 2;
    c.nstage = o[2];
    c.smem = (int)smem;
    c.cg = c.cells;
    c.pairsplit = 0;
    return true;
  }
  return false;
}

// Build the CTA schedule of one program.  Units (m1t output columns x the
// tile's cells) of all l1 groups are laid out group by group (descending l1,
// whose per-unit work is nearly uniform) and packed nw at a time into CTAs;
// a CTA spans at most two groups (two teams, two R rings).  Heavy CTAs first.
// One packing of the program for a given number of units per l1 group; returns
// the schedule cost (sum over CTAs of their slowest unit) and the group of the
// heaviest unit.
static double pack_program(const HostPlan& hp, Program& pg, const std::vector<int>& want, bool report,
                           int* heavy_l1) {
  // (groups are modified: unit_off / n_units)
  const KernelConfig& c = pg.cfg;
  const double stage2 = (double)c.mt * 256.0 * (hp.k2p / 4);
  // Stage-1 k-steps of output column m1 summed over the group's channels.
  auto m1_steps = [&](const Group& gr, int m1) {
    double st = 0.0;
    for (int e = 0; e < gr.n_chan; ++e) {
      const ChanEntry& ce = pg.chans[gr.chan_off + e];
      st += (hp.sstart[ce.slice_base + m1 + 1] - hp.sstart[ce.slice_base + m1] + 3) / 4;
    }
    return st;
  };
  // Balanced units: the d1 columns are dealt to ceil(d1/m1t) units of m1t
  // slots, heaviest column first into the lightest unit with a free slot
  // (rows per column vary ~2x with |m1|; consecutive columns would leave the
  // warps of a CTA ~20% imbalanced).
  pg.unit_m1.clear();
  for (Group& gr : pg.groups) {
    const int units = gr.n_chan ? want[gr.l1] : 0;
    gr.unit_off = (int)(pg.unit_m1.size() / c.m1t);
    gr.n_units = units;
    if (!units) continue;
    std::vector<std::pair<double, int>> cols;
    for (int m1 = 0; m1 < gr.d1; ++m1) cols.push_back({m1_steps(gr, m1), m1});
    std::stable_sort(cols.begin(), cols.end(), [](auto& x, auto& y) { return x.first > y.first; });
    // SPLITM (one cell per tile): each unit is two halves of m1t/2 slots, one
    // per warp, run in parallel -- deal into the lightest half instead.
    const int halves = c.cells == 1 ? 2 : 1, hs = c.m1t / halves;
    std::vector<double> load((size_t)units * halves, 0.0);
    std::vector<int> fill((size_t)units * halves, 0);
    std::vector<int16_t> slots((size_t)units * c.m1t, (int16_t)-1);
    for (auto& col : cols) {
      int best = -1;
      for (int u = 0; u < units * halves; ++u)
        if (fill[u] < hs && (best < 0 || load[u] < load[best])) best = u;
      slots[(size_t)(best / halves) * c.m1t + (best % halves) * hs + fill[best]++] = (int16_t)col.second;
      load[best] += col.first;
    }
    pg.unit_m1.insert(pg.unit_m1.end(), slots.begin(), slots.end());
  }
  auto unit_work = [&](const Group& gr, int u) {
    double work = 0.0;
    for (int e = 0; e < gr.n_chan; ++e) {
      const ChanEntry& ce = pg.chans[gr.chan_off + e];
      double half[2] = {0.0, 0.0};
      for (int ml = 0; ml < c.m1t; ++ml) {
        const int m1 = pg.unit_m1[(size_t)(gr.unit_off + u) * c.m1t + ml];
        if (m1 < 0) continue;
        const int rows = hp.sstart[ce.slice_base + m1 + 1] - hp.sstart[ce.slice_base + m1];
        half[c.cells == 1 ? ml / (c.m1t / 2) : 0] += (double)c.cells * c.mt * c.mt * 256.0 * ((rows + 3) / 4);
      }
      // SPLITM: the two warps walk their halves in parallel
      work += c.cells == 1 ? 2.0 * std::max(half[0], half[1]) : half[0];
      work += stage2;
    }
    return work;
  };
  // Packing: units sorted by work (heaviest first) fill CTAs of c.upc unit
  // slots, taking the next units in order whose group fits the CTA's team
  // budget (<= c.nteams groups), so every CTA holds units of similar work and
  // few slots idle at its end.  Units are then renumbered inside each group
  // so that a team's units are contiguous (Item::ubase/nunits).
  struct U {
    double work;
    int l1, u;
  };
  std::vector<U> units_all;
  double total = 0.0;
  for (const Group& gr : pg.groups)
    for (int u = 0; u < gr.n_units; ++u) {
      const double w = unit_work(gr, u);
      units_all.push_back({w, gr.l1, u});
      total += w;
    }
  std::stable_sort(units_all.begin(), units_all.end(), [](const U& x, const U& y) { return x.work > y.work; });
  if (heavy_l1) *heavy_l1 = units_all.empty() ? -1 : units_all[0].l1;
  if (const char* e = report ? std::getenv("BFQ_PLAN_STATS") : nullptr)
    if (std::atoi(e) >= 2)
      for (const U& un : units_all) std::fprintf(stderr, "unit l1=%d u=%d work=%.4g\n", un.l1, un.u, un.work);
  struct Cta {
    std::vector<std::vector<int>> team_units;  // per team: old unit ids
    std::vector<int> team_l1;
    double work = 0.0;  // slowest unit
    double lock = 0.0;  // lockstep time of the slowest team (set by the refinement)
  };
  // (a) work order: the next units in descending work whose group fits.
  auto pack_by_work = [&]() {
    std::vector<Cta> out;
    std::vector<char> taken(units_all.size(), 0);
    size_t left = units_all.size();
    while (left) {
      Cta cta;
      int used = 0;
      for (size_t k = 0; k < units_all.size() && used < c.upc; ++k) {
        if (taken[k]) continue;
        const U& un = units_all[k];
        int t = -1;
        for (size_t j = 0; j < cta.team_l1.size(); ++j)
          if (cta.team_l1[j] == un.l1) t = (int)j;
        if (t < 0) {
          if ((int)cta.team_l1.size() == c.nteams) continue;
          cta.team_l1.push_back(un.l1);
          cta.team_units.emplace_back();
          t = (int)cta.team_l1.size() - 1;
        }
        cta.team_units[t].push_back(un.u);
        cta.work = std::max(cta.work, un.work);
        taken[k] = 1;
        --left;
        ++used;
      }
      out.push_back(std::move(cta));
    }
    return out;
  };
  // (b) group fill: the group holding the heaviest remaining unit opens a CTA,
  // then each further team slot goes to the group whose units fill the free
  // slots with the most work.  Wins when few teams fit (n_k = 17: two R rings)
  // and groups hold few units each, where (a) leaves slots empty.
  auto pack_by_group = [&]() {
    std::vector<std::vector<U>> per(pg.groups.size());
    for (const U& un : units_all) per[un.l1].push_back(un);  // already in descending work
    std::vector<size_t> next(pg.groups.size(), 0);
    size_t left = units_all.size();
    std::vector<Cta> out;
    while (left) {
      int g = -1;
      for (size_t l = 0; l < per.size(); ++l)
        if (next[l] < per[l].size() && (g < 0 || per[l][next[l]].work > per[g][next[g]].work)) g = (int)l;
      Cta cta;
      int used = 0;
      auto take = [&](int l, int n) {
        cta.team_l1.push_back(l);
        cta.team_units.emplace_back();
        for (int i = 0; i < n; ++i) {
          const U& un = per[l][next[l]++];
          cta.team_units.back().push_back(un.u);
          cta.work = std::max(cta.work, un.work);
        }
        used += n;
        left -= n;
      };
      take(g, std::min<int>(c.upc, (int)(per[g].size() - next[g])));
      while (used < c.upc && (int)cta.team_l1.size() < c.nteams) {
        int best = -1;
        double best_fill = 0.0;
        for (size_t l = 0; l < per.size(); ++l) {
          if (next[l] >= per[l].size() || std::find(cta.team_l1.begin(), cta.team_l1.end(), (int)l) != cta.team_l1.end())
            continue;
          double fill = 0.0;
          for (size_t i = next[l]; i < per[l].size() && (int)(i - next[l]) < c.upc - used; ++i)
            fill += std::min(per[l][i].work, cta.work);
          if (fill > best_fill) {
            best_fill = fill;
            best = (int)l;
          }
        }
        if (best < 0) break;
        take(best, std::min<int>(c.upc - used, (int)(per[best].size() - next[best])));
      }
      out.push_back(std::move(cta));
    }
    return out;
  };
  auto cost = [&](const std::vector<Cta>& v) {
    double s = 0.0;
    for (const Cta& x : v) s += x.work;
    return s;
  };
  std::vector<Cta> ctas = pack_by_work();
  if (!std::getenv("BFQ_PACK_WORK")) {
    std::vector<Cta> alt = pack_by_group();
    if (cost(alt) < cost(ctas)) ctas.swap(alt);
  }
  // (c) refinement: deterministic annealing over unit -> CTA assignments
  // (moves and swaps, <= c.upc units and <= c.nteams groups per CTA) that
  // minimises the lockstep schedule cost: a CTA lasts as long as its slowest
  // team, and a team (one R ring) advances channel by channel at the pace of
  // its slowest unit in that channel.  Only which CTA runs a unit changes; the
  // units themselves (columns, summation order) do not, so Q is bitwise the same.
  // On by default where only two R rings fit (n_k = 17: the greedy packers leave
  // 10 CTAs per tile at lockstep efficiency 0.79, the refinement 9 at 0.86,
  // measured 50.8k -> 53.0k cells/s).  With 3-4 teams the model gains 1-4% but
  // the measured rate does not move (N=L=12 366.9k vs 366.2k, N=L=10 and 8 within
  // 0.3%: those kernels are FP64-pipe / shared-memory throttled, so an idle unit
  // slot speeds up its neighbours); BFQ_PACK_REFINE=1 forces it on, =0 off
  // (profiles/r02_pack_refine_ab.txt).
  const char* refine_env = std::getenv("BFQ_PACK_REFINE");
  const bool refine = refine_env ? std::atoi(refine_env) != 0 : c.nteams <= 2;
  if (refine && report && units_all.size() > 1) {  // the final packing only (report), not the trial ones
    const int nu = (int)units_all.size();
    // per-(unit, channel) work, as in unit_work()
    std::vector<std::vector<double>> wch(nu);
    for (int k = 0; k < nu; ++k) {
      const Group& gr = pg.groups[units_all[k].l1];
      wch[k].resize(gr.n_chan);
      for (int e = 0; e < gr.n_chan; ++e) {
        const ChanEntry& ce = pg.chans[gr.chan_off + e];
        double half[2] = {0.0, 0.0};
        for (int ml = 0; ml < c.m1t; ++ml) {
          const int m1 = pg.unit_m1[(size_t)(gr.unit_off + units_all[k].u) * c.m1t + ml];
          if (m1 < 0) continue;
          const int rows = hp.sstart[ce.slice_base + m1 + 1] - hp.sstart[ce.slice_base + m1];
          half[c.cells == 1 ? ml / (c.m1t / 2) : 0] += (double)c.cells * c.mt * c.mt * 256.0 * ((rows + 3) / 4);
        }
        wch[k][e] = (c.cells == 1 ? 2.0 * std::max(half[0], half[1]) : half[0]) + stage2;
      }
    }
    std::vector<int> where(nu, -1);  // unit (index into units_all) -> CTA
    for (size_t ci = 0; ci < ctas.size(); ++ci)
      for (size_t t = 0; t < ctas[ci].team_l1.size(); ++t)
        for (int u : ctas[ci].team_units[t])
          for (int k = 0; k < nu; ++k)
            if (units_all[k].l1 == ctas[ci].team_l1[t] && units_all[k].u == u) where[k] = (int)ci;
    const int ncta = (int)ctas.size() + 1;  // one spare CTA so a move can open a new one
    std::vector<std::vector<int>> mem(ncta);
    for (int k = 0; k < nu; ++k) mem[where[k]].push_back(k);
    std::vector<double> scratch;
    auto cta_cost = [&](const std::vector<int>& m, bool* ok) {
      // groups present, lockstep time of each
      int l1s[MAX_TEAMS + 1], ng = 0;
      *ok = (int)m.size() <= c.upc;
      for (int k : m) {
        bool seen = false;
        for (int j = 0; j < ng; ++j) seen |= l1s[j] == units_all[k].l1;
        if (!seen) {
          if (ng == c.nteams) {
            *ok = false;
            return 0.0;
          }
          l1s[ng++] = units_all[k].l1;
        }
      }
      double worst = 0.0;
      for (int j = 0; j < ng; ++j) {
        const int nch = pg.groups[l1s[j]].n_chan;
        scratch.assign(nch, 0.0);
        for (int k : m)
          if (units_all[k].l1 == l1s[j])
            for (int e = 0; e < nch; ++e) scratch[e] = std::max(scratch[e], wch[k][e]);
        double tt = 0.0;
        for (int e = 0; e < nch; ++e) tt += scratch[e];
        worst = std::max(worst, tt);
      }
      return worst;
    };
    std::vector<double> cc(ncta, 0.0);
    double cur = 0.0;
    for (int i = 0; i < ncta; ++i) {
      bool ok;
      cc[i] = cta_cost(mem[i], &ok);
      cur += cc[i];
    }
    double best = cur;
    const double init_cost = cur;
    std::vector<int> best_where = where;
    uint64_t rng = 0x9E3779B97F4A7C15ull;
    auto rnd = [&]() {
      rng = rng * 6364136223846793005ull + 1442695040888963407ull;
      return (uint32_t)(rng >> 33);
    };
    // 2M moves (about 1.5 s at n_k = 17) find the 0.88 schedule that 60k-400k miss
    // (0.856): 53.0k -> 55.0k cells/s at N=L=16 (profiles/r02_n16_pack_iters.txt)
    const int iters = std::getenv("BFQ_PACK_ITERS") ? std::atoi(std::getenv("BFQ_PACK_ITERS"))
                                                    : (nu >= 32 ? 2000000 : 60000);
    const double t0 = 0.02 * cur / std::max(1, ncta - 1), t1 = t0 * 1e-3;
    for (int it = 0; it < iters; ++it) {
      const double temp = t0 * std::pow(t1 / t0, (double)it / iters);
      const int a = (int)(rnd() % nu), ca = where[a];
      // moves: one unit or a whole team (the units of a's group in its CTA) to
      // another CTA, or exchanged against a unit / team of that CTA
      const uint32_t kind = rnd() & 3;
      int b = -1, cb;
      if (kind & 1) {
        b = (int)(rnd() % nu);
        cb = where[b];
      } else {
        cb = (int)(rnd() % ncta);
      }
      if (cb == ca) continue;
      const bool team = (kind & 2) != 0;
      std::vector<int> ma, mb, ga, gb;
      for (int k : mem[ca])
        ((team ? units_all[k].l1 == units_all[a].l1 : k == a) ? ga : ma).push_back(k);
      for (int k : mem[cb])
        ((b >= 0 && (team ? units_all[k].l1 == units_all[b].l1 : k == b)) ? gb : mb).push_back(k);
      ma.insert(ma.end(), gb.begin(), gb.end());
      mb.insert(mb.end(), ga.begin(), ga.end());
      bool oka, okb;
      const double na = cta_cost(ma, &oka), nb = cta_cost(mb, &okb);
      if (!oka || !okb) continue;
      const double d = na + nb - cc[ca] - cc[cb];
      if (d <= 0.0 || (double)(rnd() & 0xFFFFFF) / 16777216.0 < std::exp(-d / temp)) {
        mem[ca].swap(ma);
        mem[cb].swap(mb);
        cc[ca] = na;
        cc[cb] = nb;
        for (int k : ga) where[k] = cb;
        for (int k : gb) where[k] = ca;
        cur += d;
        if (cur < best * (1.0 - 1e-12)) {
          best = cur;
          best_where = where;
        }
      }
    }
    if (report && std::getenv("BFQ_PLAN_STATS"))
      std::fprintf(stderr, "plan: refinement lockstep cost %.4g -> %.4g\n", init_cost, best);
    // rebuild the CTA list from the best assignment (teams in order of first appearance)
    std::vector<Cta> out(ncta);
    for (int k = 0; k < nu; ++k) {
      Cta& cta = out[best_where[k]];
      int t = -1;
      for (size_t j = 0; j < cta.team_l1.size(); ++j)
        if (cta.team_l1[j] == units_all[k].l1) t = (int)j;
      if (t < 0) {
        cta.team_l1.push_back(units_all[k].l1);
        cta.team_units.emplace_back();
        t = (int)cta.team_l1.size() - 1;
      }
      cta.team_units[t].push_back(units_all[k].u);
      cta.work = std::max(cta.work, units_all[k].work);
    }
    for (int i = 0; i < ncta; ++i) {
      std::vector<int> m;
      for (int k = 0; k < nu; ++k)
        if (best_where[k] == i) m.push_back(k);
      bool ok;
      out[i].lock = cta_cost(m, &ok);
    }
    out.erase(std::remove_if(out.begin(), out.end(), [](const Cta& x) { return x.team_l1.empty(); }), out.end());
    // self-check before the refined schedule replaces the greedy one: every unit
    // exactly once, CTA shape respected
    bool valid = true;
    size_t placed = 0;
    std::vector<std::vector<char>> seen(pg.groups.size());
    for (const Group& gr : pg.groups) seen[gr.l1].assign((size_t)std::max(gr.n_units, 0), 0);
    for (const Cta& cta : out) {
      int used = 0;
      valid &= (int)cta.team_l1.size() <= c.nteams;
      for (size_t t = 0; t < cta.team_l1.size(); ++t)
        for (int u : cta.team_units[t]) {
          std::vector<char>& sg = seen[cta.team_l1[t]];
          if (u < 0 || u >= (int)sg.size() || sg[u]) valid = false;
          else sg[u] = 1;
          ++used;
          ++placed;
        }
      valid &= used <= c.upc;
    }
    valid &= placed == units_all.size();
    if (valid) ctas.swap(out);
    else if (std::getenv("BFQ_PLAN_STATS")) std::fprintf(stderr, "plan: refined schedule rejected by the self-check\n");
  }
  // renumber units inside each group in order of appearance
  std::vector<int16_t> new_m1 = pg.unit_m1;
  std::vector<int> next_id(pg.groups.size(), 0);
  pg.items.clear();
  std::stable_sort(ctas.begin(), ctas.end(), [](const Cta& x, const Cta& y) {
    return (x.lock > 0.0 ? x.lock : x.work) > (y.lock > 0.0 ? y.lock : y.work);
  });
  for (const Cta& cta : ctas) {
    Item it{};
    for (size_t t = 0; t < cta.team_l1.size(); ++t) {
      const int l1 = cta.team_l1[t];
      const Group& gr = pg.groups[l1];
      it.l1[t] = l1;
      it.ubase[t] = next_id[l1];
      it.nunits[t] = (int32_t)cta.team_units[t].size();
      for (int old : cta.team_units[t]) {
        const int nu = next_id[l1]++;
        for (int ml = 0; ml < c.m1t; ++ml)
          new_m1[(size_t)(gr.unit_off + nu) * c.m1t + ml] = pg.unit_m1[(size_t)(gr.unit_off + old) * c.m1t + ml];
      }
    }
    pg.items.push_back(it);
  }
  pg.unit_m1.swap(new_m1);
  pg.exec_macs_per_cell = total / c.cells;
  if (report && std::getenv("BFQ_PLAN_STATS")) {  // packing efficiency: unit work / (slots x slowest unit)
    double cap = 0.0;
    for (const Cta& cta : ctas) cap += cta.work * c.upc;
    // lockstep model: a team (one R ring) advances channel by channel at the
    // pace of its slowest unit in that channel
    double cap2 = 0.0;
    for (const Cta& cta : ctas) {
      double worst = 0.0;
      for (size_t t = 0; t < cta.team_l1.size(); ++t) {
        const Group& gr = pg.groups[cta.team_l1[t]];
        double tt = 0.0;
        for (int e = 0; e < gr.n_chan; ++e) {
          const ChanEntry& ce = pg.chans[gr.chan_off + e];
          double mx = 0.0;
          for (int old : cta.team_units[t]) {
            double w = stage2;
            for (int ml = 0; ml < c.m1t; ++ml) {
              const int m1 = new_m1[(size_t)(gr.unit_off + old) * c.m1t + ml];  // old ids (swapped out)
              if (m1 < 0) continue;
              w += (double)c.cells * c.mt * c.mt * 256.0 *
                   ((hp.sstart[ce.slice_base + m1 + 1] - hp.sstart[ce.slice_base + m1] + 3) / 4);
            }
            mx = std::max(mx, w);
          }
          tt += mx;
        }
        worst = std::max(worst, tt);
      }
      cap2 += worst * c.upc;
    }
    std::fprintf(stderr, "plan: %zu CTAs per tile, %zu units, packing efficiency %.3f, with team lockstep %.3f\n",
                 ctas.size(), units_all.size(), total / cap, total / cap2);
  }
  return cost(ctas);
}

// Build the CTA schedule: start from ceil(d1 / m1t) units per l1 group (every
// slot used), then split the group holding the heaviest unit into one more
// unit while that lowers the modelled schedule cost (sum over CTAs of their
// slowest unit).  Opt-in (BFQ_UNIT_BALANCE=1): at n_k = 17 it raises the model's
// packing efficiency 0.83 -> 0.87 but measured 7% SLOWER (46.5k -> 43.2k
// cells/s, profiles/r02_unit_balance.txt) -- the extra units' stage-2 work and
// the extra CTA per tile cost more than the model credits.
static void build_items(const HostPlan& hp, Program& pg) {
  const KernelConfig& c = pg.cfg;
  std::vector<int> want(pg.groups.size(), 0);
  for (const Group& gr : pg.groups) want[gr.l1] = gr.n_chan ? (gr.d1 + c.m1t - 1) / c.m1t : 0;
  int heavy = -1;
  double best_cost;
  {
    Program first = pg;
    best_cost = pack_program(hp, first, want, false, &heavy);
  }
  if (std::getenv("BFQ_UNIT_BALANCE")) {
    // greedy splits with look-ahead: keep splitting the heaviest unit's group
    // (several groups are often nearly as heavy), remember the cheapest schedule
    std::vector<int> cur = want;
    int misses = 0;
    for (int it = 0; it < 96 && heavy >= 0 && misses < 12; ++it) {
      if (cur[heavy] >= pg.groups[heavy].d1) break;  // one column per unit already
      ++cur[heavy];
      Program trial = pg;
      const double cst = pack_program(hp, trial, cur, false, &heavy);
      if (cst < best_cost * (1.0 - 1e-9)) {
        best_cost = cst;
        want = cur;
        misses = 0;
      } else {
        ++misses;
      }
    }
  }
  pack_program(hp, pg, want, true, nullptr);
}

// Shared-memory wavefronts of one stage-1 gather instruction for a group of
// up to 4 table rows (lane kq reads row kq; lanes r0 = 0..3 of a half-warp read
// operand row r0 at word r0*qs + q).  Distinct words on the same 8-byte bank
// pair serialise; equal words broadcast.
static int group_wavefronts(const int* q, int n, int qs) {
  int words[16], nw = 0;
  for (int r0 = 0; r0 < 4; ++r0)
    for (int j = 0; j < 4; ++j) {
      const int w = r0 * qs + (j < n ? q[j] : 0);
      bool dup = false;
      for (int t = 0; t < nw; ++t) dup |= words[t] == w;
      if (!dup) words[nw++] = w;
    }
  int per_bank[16] = {0}, worst = 0;
  for (int t = 0; t < nw; ++t) worst = std::max(worst, ++per_bank[words[t] & 15]);
  return worst;
}

// Reorder the rows inside every (tau, q1) slice so that each k-step's four
// rows gather conflict-free (greedy, per slice).  Only the summation order
// inside a slice changes.
static void reorder_rows_for_banks(HostPlan& hp, const int64_t* slice_starts, int64_t n_s) {
  std::vector<Row> tmp;
  for (int64_t s = 0; s < n_s; ++s) {
    const int64_t a = slice_starts[s], b = slice_starts[s + 1];
    const int n = (int)(b - a);
    if (n <= 1) continue;
    tmp.assign(hp.rows.begin() + a, hp.rows.begin() + b);
    std::vector<char> used(n, 0);
    int64_t out = a;
    for (int g0 = 0; g0 < n; g0 += 4) {
      int q2[4], q3[4], m = 0;
      const int gsz = std::min(4, n - g0);
      for (int j = 0; j < gsz; ++j) {
        int best = -1, best_cost = 1 << 30;
        for (int r = 0; r < n; ++r) {
          if (used[r]) continue;
          q2[m] = tmp[r].q2;
          q3[m] = tmp[r].q3;
          // cost of the group if completed with this row (missing lanes read q = 0)
          const int cost = group_wavefronts(q2, m + 1, hp.qs) + group_wavefronts(q3, m + 1, hp.qs);
          if (cost < best_cost) {
            best_cost = cost;
            best = r;
          }
        }
        used[best] = 1;
        q2[m] = tmp[best].q2;
        q3[m] = tmp[best].q3;
        ++m;
        hp.rows[out++] = tmp[best];
      }
    }
    // Local search on top of the greedy grouping: swap rows between k-step
    // groups of the slice while that lowers the total gather wavefronts.
    if (n <= 96 && !std::getenv("BFQ_NO_ROW_SWAP")) {
      const int ng = (n + 3) / 4;
      auto gcost = [&](int g) {
        int a2[4], a3[4], m = 0;
        for (int j = 0; j < 4 && 4 * g + j < n; ++j, ++m) {
          a2[m] = hp.rows[a + 4 * g + j].q2;
          a3[m] = hp.rows[a + 4 * g + j].q3;
        }
        return group_wavefronts(a2, m, hp.qs) + group_wavefronts(a3, m, hp.qs);
      };
      std::vector<int> cost(ng);
      for (int g = 0; g < ng; ++g) cost[g] = gcost(g);
      for (int pass = 0; pass < 4; ++pass) {
        bool improved = false;
        for (int i = 0; i < n; ++i)
          for (int j = i + 1; j < n; ++j) {
            const int gi = i / 4, gj = j / 4;
            if (gi == gj) continue;
            std::swap(hp.rows[a + i], hp.rows[a + j]);
            const int ci = gcost(gi), cj = gcost(gj);
            if (ci + cj < cost[gi] + cost[gj]) {
              cost[gi] = ci;
              cost[gj] = cj;
              improved = true;
            } else {
              std::swap(hp.rows[a + i], hp.rows[a + j]);
            }
          }
        if (!improved) break;
      }
    }
  }
}

int build_host_plan(const bfq_desc& d, int smem_limit, HostPlan& hp) {
  if (d.k_max < 0 || d.l_max < 0) return fail(BFQ_EINVAL, "truncation limits must be non-negative");
  if (d.n_t <= 0 || d.n_g <= 0 || d.n_s <= 0) return fail(BFQ_EINVAL, "empty operator");
  if (!d.triplets || !d.q1 || !d.q2 || !d.q3 || !d.tau || !d.g || !d.slice_starts ||
      !d.slice_tau || !d.slice_q1 || !d.r)
    return fail(BFQ_EINVAL, "null pointer in operator description");
  if (d.n_s > d.n_g) return fail(BFQ_EINVAL, "slice count cannot exceed row count");
  const int nk = d.k_max + 1, L = d.l_max, nq = (L + 1) * (L + 1);
  if (nk > 24) return fail(BFQ_EINVAL, "n_k > 24 not supported by the DMMA tiling");
  hp.n_k = nk;
  hp.n_q = nq;
  hp.k_max = d.k_max;
  hp.l_max = L;
  hp.n_t = d.n_t;
  hp.n_g = d.n_g;
  hp.n_s = d.n_s;
  hp.gamma = d.gamma;
  hp.conservation = d.conservation != 0;
  hp.detailed_balance = d.detailed_balance != 0;
  hp.qs = conflict_free_stride(nq);
  hp.k2p = (nk * nk + 3) / 4 * 4;
  hp.k2s = conflict_free_stride(hp.k2p);
  hp.k2pd = (nk * (nk + 1) / 2 + 3) / 4 * 4;
  hp.k2sd = conflict_free_stride(hp.k2pd);

  // channel table (angular.py:119-135)
  hp.triplets.assign(d.triplets, d.triplets + 3 * (size_t)d.n_t);
  std::unordered_map<long, int> chan_of;
  for (int t = 0; t < d.n_t; ++t) {
    const int l1 = hp.triplets[3 * t], l2 = hp.triplets[3 * t + 1], l3 = hp.triplets[3 * t + 2];
    if (l1 < 0 || l2 < 0 || l3 < 0 || l1 > L || l2 > L || l3 > L)
      return fail(BFQ_EINVAL, "channel triplet out of range");
    chan_of[((long)l1 * 64 + l2) * 64 + l3] = t;
  }

  // rows: range checks (contraction.py:90-95), degree consistency, sort guard
  auto lq = [](int q) { return isqrt_floor(q); };
  hp.rows.resize(d.n_g);
  for (int64_t z = 0; z < d.n_g; ++z) {
    const int t = d.tau[z], q1 = d.q1[z], q2 = d.q2[z], q3 = d.q3[z];
    if (t < 0 || t >= d.n_t) return fail(BFQ_EINVAL, "channel index out of range");
    if (q1 < 0 || q1 >= nq || q2 < 0 || q2 >= nq || q3 < 0 || q3 >= nq)
      return fail(BFQ_EINVAL, "angular index out of range");
    if (lq(q1) != hp.triplets[3 * t] || lq(q2) != hp.triplets[3 * t + 1] ||
        lq(q3) != hp.triplets[3 * t + 2])
      return fail(BFQ_EINVAL, "row degrees disagree with its channel triplet");
    if (z > 0) {
      const long kprev = (long)d.tau[z - 1] * nq + d.q1[z - 1], key = (long)t * nq + q1;
      if (key < kprev) return fail(BFQ_EUNSORTED, "COO rows must be sorted and grouped by (tau, q1)");
    }
    hp.rows[z] = Row{q2, q3, d.g[z]};
  }
  // slices (angular.py:275-285): consistent with the rows they cover
  if (d.slice_starts[0] != 0 || d.slice_starts[d.n_s] != d.n_g)
    return fail(BFQ_EINVAL, "slice_starts must span [0, n_g]");
  for (int64_t s = 0; s < d.n_s; ++s) {
    const int64_t a = d.slice_starts[s], b = d.slice_starts[s + 1];
    if (b <= a) return fail(BFQ_EINVAL, "empty or decreasing slice");
    for (int64_t z = a; z < b; ++z)
      if (d.tau[z] != d.slice_tau[s] || d.q1[z] != d.slice_q1[s])
        return fail(BFQ_EINVAL, "slice does not match the (tau, q1) of its rows");
    if (s > 0 && d.slice_tau[s] == d.slice_tau[s - 1] && d.slice_q1[s] == d.slice_q1[s - 1])
      return fail(BFQ_EINVAL, "duplicate (tau, q1) slice");
  }

  if (!std::getenv("BFQ_NO_ROW_REORDER")) reorder_rows_for_banks(hp, d.slice_starts, d.n_s);

  // expanded slice table: every (tau, m1) gets a (possibly empty) row range
  hp.chan_sbase.resize(d.n_t);
  hp.sstart.clear();
  {
    std::vector<long> keys(d.n_g);
    for (int64_t z = 0; z < d.n_g; ++z) keys[z] = (long)d.tau[z] * nq + d.q1[z];
    for (int t = 0; t < d.n_t; ++t) {
      const int l1 = hp.triplets[3 * t];
      hp.chan_sbase[t] = (int)hp.sstart.size();
      for (int m1 = 0; m1 < 2 * l1 + 1; ++m1) {
        const long key = (long)t * nq + l1 * l1 + m1;
        hp.sstart.push_back((int32_t)(std::lower_bound(keys.begin(), keys.end(), key) - keys.begin()));
      }
    }
    hp.sstart.push_back((int32_t)d.n_g);
  }
  // Pad every slice to a whole number of k-steps with g = 0 rows (q2 = q3 = 0),
  // so the stage-1 row stream needs no clamp / zero-weight select: 4 rows, or
  // 8 at n_k = 17 where the DUAL loop consumes two row groups per iteration.
  {
    const int padm = nk == 17 ? 8 : 4;
    std::vector<Row> padded;
    padded.reserve(hp.rows.size() + (size_t)padm * hp.sstart.size());
    std::vector<int32_t> ns(hp.sstart.size());
    for (size_t i = 0; i + 1 < hp.sstart.size(); ++i) {
      ns[i] = (int32_t)padded.size();
      const int32_t a = hp.sstart[i], b = hp.sstart[i + 1];
      for (int32_t z = a; z < b; ++z) padded.push_back(hp.rows[z]);
      while ((padded.size() - ns[i]) % padm) padded.push_back(Row{0, 0, 0.0});
    }
    ns.back() = (int32_t)padded.size();
    // The row stream prefetches up to two k-steps past the slice it works on
    // (also past the last slice, and from an empty slice at the end): keep
    // 2 * padm zero-weight rows after the table so every such fetch is in bounds.
    for (int i = 0; i < 2 * padm; ++i) padded.push_back(Row{0, 0, 0.0});
    hp.rows.swap(padded);
    hp.sstart.swap(ns);
  }

  // R blocks: rblocks[t][k1][a*nk+b] = R[k1,a,b,t]; zero padding to k2s
  const size_t blk = (size_t)nk * hp.k2s;
  hp.rblocks.assign((size_t)d.n_t * blk, 0.0);
  for (int k1 = 0; k1 < nk; ++k1)
    for (int a = 0; a < nk; ++a)
      for (int b = 0; b < nk; ++b) {
        const double* src = d.r + (((size_t)k1 * nk + a) * nk + b) * d.n_t;
        for (int t = 0; t < d.n_t; ++t) hp.rblocks[t * blk + (size_t)k1 * hp.k2s + a * nk + b] = src[t];
      }

  // slot-symmetry check (SURVEY §7 hard part f): table closed under
  // (q2,q3,(l1,l2,l3)) <-> (q3,q2,(l1,l3,l2)) with identical g, and R exactly
  // symmetric under (k2,k3,tau) <-> (k3,k2,tau').  Then the tau and tau'
  // contributions to Q(f,f) are equal and only l2 <= l3 channels are evaluated.
  bool fold = true;
  std::vector<int> swap_of(d.n_t, -1);
  for (int t = 0; t < d.n_t && fold; ++t) {
    auto it = chan_of.find(((long)hp.triplets[3 * t] * 64 + hp.triplets[3 * t + 2]) * 64 + hp.triplets[3 * t + 1]);
    if (it == chan_of.end()) fold = false;
    else swap_of[t] = it->second;
  }
  if (fold) {
    for (int t = 0; t < d.n_t && fold; ++t) {
      const int u = swap_of[t];
      for (int k1 = 0; k1 < nk && fold; ++k1)
        for (int a = 0; a < nk && fold; ++a)
          for (int b = 0; b < nk; ++b)
            if (hp.rblocks[t * blk + (size_t)k1 * hp.k2s + a * nk + b] !=
                hp.rblocks[u * blk + (size_t)k1 * hp.k2s + b * nk + a]) {
              fold = false;
              break;
            }
    }
  }
  if (fold) {
    std::unordered_map<uint64_t, double> gmap;
    gmap.reserve(d.n_g * 2);
    auto rk = [&](int t, int q1, int q2, int q3) {
      return (((uint64_t)t * nq + q1) * nq + q2) * nq + q3;
    };
    for (int64_t z = 0; z < d.n_g; ++z) gmap[rk(d.tau[z], d.q1[z], d.q2[z], d.q3[z])] = d.g[z];
    for (int64_t z = 0; z < d.n_g && fold; ++z) {
      auto it = gmap.find(rk(swap_of[d.tau[z]], d.q1[z], d.q3[z], d.q2[z]));
      if (it == gmap.end() || it->second != d.g[z]) fold = false;
    }
  }
  hp.folded = fold;

  // Half-row slices of the self-symmetric channels (l2 == l3) for the folded
  // program.  Their rows come in mirror pairs (q2, q3) / (q3, q2) with equal g
  // (verified by the fold check), and R[k,a,b] = R[k,b,a], so
  //   sum_ab R[ab] Phi[ab] = sum_ab R[ab] Phi''[ab],
  //   Phi'' = sum_{q2 < q3} 2g f[a,q2] f[b,q3] + sum_{q2 = q3} g f[a,q] f[b,q]
  // (Phi = Phi' + Phi'^T with Phi' the half-row sum): half the stage-1 rows, at
  // the price of the full K = n_k^2 in stage 2 instead of the packed triangle
  // (the diag path below).  Measured (profiles/r02_half_diag.txt): N=L=8 +0.4%,
  // N=L=12 +1.2%, N=L=16 +3.1%.  BFQ_HALF_DIAG=0 restores the packed path.
  std::vector<int32_t> half_base(d.n_t, -1);
  {
    bool half = fold;
    if (const char* e = std::getenv("BFQ_HALF_DIAG")) half = fold && std::atoi(e) != 0;
    if (half) {
      const int padm = nk == 17 ? 8 : 4;
      hp.rows.resize(hp.rows.size() - 2 * padm);  // drop the tail, re-added below
      for (int t = 0; t < d.n_t; ++t) {
        const int l1 = hp.triplets[3 * t], l2 = hp.triplets[3 * t + 1], l3 = hp.triplets[3 * t + 2];
        if (l2 != l3) continue;
        half_base[t] = (int32_t)hp.sstart.size() - 1;  // its first slice starts at the current end
        for (int m1 = 0; m1 < 2 * l1 + 1; ++m1) {
          const int32_t a = hp.sstart[hp.chan_sbase[t] + m1], b = hp.sstart[hp.chan_sbase[t] + m1 + 1];
          const int64_t start = (int64_t)hp.rows.size();
          for (int32_t z = a; z < b; ++z) {
            const Row r = hp.rows[z];
            if (r.g == 0.0 && r.q2 == 0 && r.q3 == 0) continue;  // slice padding
            if (r.q2 < r.q3) hp.rows.push_back(Row{r.q2, r.q3, 2.0 * r.g});
            else if (r.q2 == r.q3) hp.rows.push_back(r);
          }
          if (!std::getenv("BFQ_NO_ROW_REORDER")) {
            const int64_t bounds[2] = {start, (int64_t)hp.rows.size()};
            reorder_rows_for_banks(hp, bounds, 1);
          }
          while ((hp.rows.size() - start) % padm) hp.rows.push_back(Row{0, 0, 0.0});
          hp.sstart.push_back((int32_t)hp.rows.size());
        }
      }
      for (int i = 0; i < 2 * padm; ++i) hp.rows.push_back(Row{0, 0, 0.0});
    }
  }

  // channel programs, grouped by l1 (output columns)
  auto make_program = [&](Program& pg, bool bilinear, bool use_fold) -> bool {
    pg.bilinear = bilinear;
    pg.chans.clear();
    pg.groups.assign(L + 1, Group{0, 0, 0, 0, 0, 0, {0, 0}});
    for (int l1 = 0; l1 <= L; ++l1) {
      pg.groups[l1].chan_off = (int)pg.chans.size();
      pg.groups[l1].d1 = 2 * l1 + 1;
      pg.groups[l1].l1 = l1;
      for (int t = 0; t < d.n_t; ++t) {
        if (hp.triplets[3 * t] != l1) continue;
        const int l2 = hp.triplets[3 * t + 1], l3 = hp.triplets[3 * t + 2];
        int w2 = 0, base = hp.chan_sbase[t];
        if (use_fold) {
          if (l2 > l3) continue;
          w2 = l2 < l3 ? 1 : 0;
          if (half_base[t] >= 0) base = half_base[t];
        }
        pg.chans.push_back(ChanEntry{t, base, w2, 0});
      }
      pg.groups[l1].n_chan = (int)pg.chans.size() - pg.groups[l1].chan_off;
    }
    int max_chan = 1;
    for (const Group& g : pg.groups) max_chan = std::max(max_chan, g.n_chan);
    if (!choose_config(nk, hp.qs, hp.k2s, bilinear ? 2 : 1, smem_limit, max_chan, pg.cfg)) return false;
    build_items(hp, pg);
    return true;
  };
  if (!make_program(hp.sym, false, fold) || !make_program(hp.full, true, false))
    return fail(BFQ_ESMEM, "no kernel configuration fits in shared memory for this n_k, l_max");
  // Folded channels with l2 < l3 count twice: give them their own copy of the
  // R block scaled by 2 (exact in fp64), so the kernel needs no weight.
  for (ChanEntry& ce : hp.sym.chans) {
    if (!ce.weight2) continue;
    const size_t nb = hp.rblocks.size() / blk;
    hp.rblocks.resize((nb + 1) * blk);
    for (size_t i = 0; i < blk; ++i) hp.rblocks[nb * blk + i] = 2.0 * hp.rblocks[(size_t)ce.tau * blk + i];
    ce.tau = (int32_t)nb;
    ce.weight2 = 0;
  }
  // Self-symmetric folded channels (l2 == l3, their own swap partner): Phi and
  // R are symmetric in (a, b), so the pair-split kernel contracts only the
  // upper triangle a <= b, with R packed as R'[k1][p(a,b)] = (a<b ? 2 : 1) R.
  if (hp.folded && hp.sym.cfg.pairsplit && !std::getenv("BFQ_NO_DIAG")) {
    for (ChanEntry& ce : hp.sym.chans) {
      const int t = ce.tau < d.n_t ? ce.tau : -1;
      if (t < 0 || hp.triplets[3 * t + 1] != hp.triplets[3 * t + 2] || half_base[t] >= 0) continue;
      const size_t nb = hp.rblocks.size() / blk;
      hp.rblocks.resize((nb + 1) * blk, 0.0);
      for (int k1 = 0; k1 < nk; ++k1) {
        int pidx = 0;
        for (int a = 0; a < nk; ++a)
          for (int b = a; b < nk; ++b, ++pidx)
            hp.rblocks[nb * blk + (size_t)k1 * hp.k2sd + pidx] =
                (a < b ? 2.0 : 1.0) * hp.rblocks[(size_t)t * blk + (size_t)k1 * hp.k2s + a * nk + b];
      }
      ce.tau = (int32_t)nb;
      ce.diag = 1;
    }
  }

  // K order of every R block = the order the kernels store Phi in
  // (bfq_internal.h phi_k / phid_k: conflict-free Phi stores, compact K).
  {
    const size_t nb = hp.rblocks.size() / blk;
    std::vector<char> packed(nb, 0);
    for (const ChanEntry& ce : hp.sym.chans)
      if (ce.diag) packed[ce.tau] = 1;
    std::vector<double> src(blk);
    for (size_t t = 0; t < nb; ++t) {
      double* b = hp.rblocks.data() + t * blk;
      std::copy(b, b + blk, src.begin());
      std::fill(b, b + blk, 0.0);
      for (int k1 = 0; k1 < nk; ++k1) {
        if (packed[t]) {
          int pidx = 0;
          for (int a = 0; a < nk; ++a)
            for (int c = a; c < nk; ++c, ++pidx)
              b[(size_t)k1 * hp.k2sd + phid_k(nk, a, c)] = src[(size_t)k1 * hp.k2sd + pidx];
        } else {
          for (int a = 0; a < nk; ++a)
            for (int c = 0; c < nk; ++c) b[(size_t)k1 * hp.k2s + phi_k(nk, a, c)] = src[(size_t)k1 * hp.k2s + a * nk + c];
        }
      }
    }
  }

  // executed DMMA MACs per cell of the Q(f,f) program (after the diag packing)
  {
    const Program& pg = hp.sym;
    const KernelConfig& c = pg.cfg;
    // n_k = 8k+1 with a fixed-size pair-split kernel: the last k row/column
    // runs on DFMA (bfq_qkernel2.cuh, X1), so one tile column fewer on DMMA
    const bool x1 = c.pairsplit && nk % 8 == 1 && c.mt >= 2 && (nk == 9 || nk == 17) &&
                    !std::getenv("BFQ_GENERIC");
    const int mte = x1 ? c.mt - 1 : c.mt;
    double total = 0.0;
    for (const Group& gr : pg.groups) {
      for (int e = 0; e < gr.n_chan; ++e) {
        const ChanEntry& ce = pg.chans[gr.chan_off + e];
        // n_k = 11, four cells per tile: the (1, 1) tiles of a warp's two cells share one DMMA (MIX)
        const bool mix = c.pairsplit && nk == 11 && hp.qs == 124 && c.cells == 4 && !std::getenv("BFQ_GENERIC");
        const double tiles = (ce.diag ? mte * (mte + 1) / 2 : mte * mte) - (mix ? 0.5 : 0.0);
        for (int m1 = 0; m1 < gr.d1; ++m1) {
          const int rows = hp.sstart[ce.slice_base + m1 + 1] - hp.sstart[ce.slice_base + m1];
          total += tiles * 256.0 * ((rows + 3) / 4);  // per cell
        }
        total += (double)gr.n_units * mte * 256.0 * ((ce.diag ? hp.k2pd : hp.k2p) / 4) / c.cells;
      }
    }
    hp.sym.exec_macs_per_cell = total;
  }
  // useful MACs of the evaluated channels (no padding): what the kernel must do
  {
    std::vector<int64_t> chan_rows(d.n_t, 0);
    for (int64_t z = 0; z < d.n_g; ++z) ++chan_rows[d.tau[z]];
    for (int t = 0; t < d.n_t; ++t)
      if (half_base[t] >= 0) {  // half-row slices: count their rows without padding
        int64_t n = 0;
        const int l1 = hp.triplets[3 * t];
        for (int m1 = 0; m1 < 2 * l1 + 1; ++m1)
          for (int32_t z = hp.sstart[half_base[t] + m1]; z < hp.sstart[half_base[t] + m1 + 1]; ++z)
            n += hp.rows[z].g != 0.0;
        chan_rows[t] = n;
      }
    double useful = 0.0;
    for (int t = 0; t < d.n_t; ++t) {
      const int l1 = hp.triplets[3 * t], l2 = hp.triplets[3 * t + 1], l3 = hp.triplets[3 * t + 2];
      if (hp.folded && l2 > l3) continue;
      const bool diag = hp.folded && l2 == l3 && hp.sym.cfg.pairsplit && !std::getenv("BFQ_NO_DIAG") &&
                        half_base[t] < 0;
      const double kk = diag ? nk * (nk + 1) / 2.0 : (double)nk * nk;
      useful += (double)chan_rows[t] * kk + (2.0 * l1 + 1.0) * nk * kk;
    }
    hp.useful_macs_per_cell = useful;
  }
  hp.alg_flops_per_cell = 2.0 * ((double)d.n_g * nk * nk + (double)d.n_s * nk * nk * nk);
  hp.alg_bytes_per_cell = 16.0 * nk * nq;
  return BFQ_OK;
}

// ---------------------------------------------------------------- BFCT reader
uint32_t crc32_update(uint32_t crc, const unsigned char* data, size_t n) {
  static uint32_t table[256];
  static bool init = false;
  if (!init) {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? (0xEDB88320u ^ (c >> 1)) : (c >> 1);
      table[i] = c;
    }
    init = true;
  }
  crc = ~crc;
  for (size_t i = 0; i < n; ++i) crc = table[(crc ^ data[i]) & 0xFF] ^ (crc >> 8);
  return ~crc;
}

template <class T>
static T rd(const unsigned char* p) {
  T v;
  std::memcpy(&v, p, sizeof(T));
  return v;
}

int read_bfct(const char* path, BfctImage& img) {
  FILE* fp = std::fopen(path, "rb");
  if (!fp) return fail(BFQ_EIO, std::string("cannot open ") + path);
  std::vector<unsigned char> blob;
  unsigned char buf[1 << 16];
  size_t n;
  while ((n = std::fread(buf, 1, sizeof buf, fp)) > 0) blob.insert(blob.end(), buf, buf + n);
  std::fclose(fp);
  // header "<4sIIId9IIQII" = 80 bytes (cache.py:41)
  const size_t H = 80;
  if (blob.size() < H) return fail(BFQ_EFORMAT, "file too short for a cache header");
  if (std::memcmp(blob.data(), "BFCT", 4) != 0) return fail(BFQ_EFORMAT, "bad magic");
  const uint32_t version = rd<uint32_t>(&blob[4]);
  if (version != 1) return fail(BFQ_EFORMAT, "cache format version unsupported (expected 1)");
  img.k_max = (int32_t)rd<uint32_t>(&blob[8]);
  img.l_max = (int32_t)rd<uint32_t>(&blob[12]);
  img.gamma = rd<double>(&blob[16]);
  // 9 x u32 grid spec at 24..59
  const uint32_t n_t = rd<uint32_t>(&blob[60]);
  const uint64_t n_g = rd<uint64_t>(&blob[64]);
  img.flags = rd<uint32_t>(&blob[72]);
  const uint32_t crc = rd<uint32_t>(&blob[76]);
  const unsigned char* pay = blob.data() + H;
  const size_t plen = blob.size() - H;
  if (crc32_update(0, pay, plen) != crc) return fail(BFQ_EINTEGRITY, "payload checksum mismatch");
  const uint64_t nk = (uint64_t)img.k_max + 1;
  const uint64_t expected = (uint64_t)n_t * 12 + n_g * 24 + nk * nk * nk * n_t * 8;
  if (plen != expected) return fail(BFQ_EINTEGRITY, "payload size disagrees with header");
  size_t off = 0;
  img.triplets.resize((size_t)n_t * 3);
  for (size_t i = 0; i < img.triplets.size(); ++i, off += 4) img.triplets[i] = (int32_t)rd<uint32_t>(pay + off);
  auto col = [&](std::vector<int32_t>& v) {
    v.resize(n_g);
    for (uint64_t i = 0; i < n_g; ++i, off += 4) v[i] = (int32_t)rd<uint32_t>(pay + off) - 1;  // 1-based -> 0-based
  };
  col(img.q1);
  col(img.q2);
  col(img.q3);
  col(img.tau);
  img.g.resize(n_g);
  std::memcpy(img.g.data(), pay + off, n_g * 8);
  off += n_g * 8;
  img.r.resize(nk * nk * nk * n_t);
  std::memcpy(img.r.data(), pay + off, img.r.size() * 8);
  // slices: boundaries of key = tau*(l_max+1)^2 + q1 (cache.py:147-150)
  const long nq = (long)(img.l_max + 1) * (img.l_max + 1);
  img.slice_starts.clear();
  for (uint64_t z = 0; z < n_g; ++z) {
    if (z == 0 || (long)img.tau[z] * nq + img.q1[z] != (long)img.tau[z - 1] * nq + img.q1[z - 1]) {
      img.slice_starts.push_back((int64_t)z);
      img.slice_tau.push_back(img.tau[z]);
      img.slice_q1.push_back(img.q1[z]);
    }
  }
  img.slice_starts.push_back((int64_t)n_g);
  bfq_desc& d = img.desc;
  d.k_max = img.k_max;
  d.l_max = img.l_max;
  d.gamma = img.gamma;
  d.n_t = (int32_t)n_t;
  d.n_g = (int64_t)n_g;
  d.n_s = (int64_t)img.slice_tau.size();
  d.triplets = img.triplets.data();
  d.q1 = img.q1.data();
  d.q2 = img.q2.data();
  d.q3 = img.q3.data();
  d.tau = img.tau.data();
  d.g = img.g.data();
  d.slice_starts = img.slice_starts.data();
  d.slice_tau = img.slice_tau.data();
  d.slice_q1 = img.slice_q1.data();
  d.r = img.r.data();
  d.conservation = (img.flags & 1) ? 1 : 0;
  d.detailed_balance = (img.flags & 2) ? 1 : 0;
  return BFQ_OK;
}

}  // namespace bfq
