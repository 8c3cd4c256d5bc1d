// Tile plan of the bulk-copy evaluator (phx_bulk.cu): the inspector half of an
// inspector-executor SpMM.  Built once per operator on the host (the reference
// operator is immutable, linop.hpp:16-18), O(nnz), tiles in parallel.
//
// For every kPlanT-row tile the gather sources of its CSR entries are covered
// by CONTIGUOUS row ranges that the kernel stages with one cp.async.bulk copy
// each:
//   - the window [base-1, base+T+1): the tile's own rows, the diagonal and
//     every column inside it (C5's bidiagonal rows need nothing else);
//   - up to kPlanGroups offset groups: entries whose column - row offset is
//     shared by at least max(2, rows/4) rows of the tile (a 3D 7-point stencil
//     has four: +-nx and +-nx*ny), staged as the rows [base+off, base+off+T);
//   - single rows for everything else (at most kPlanMaxSingles per tile).
// Each entry gets a one-byte slot: its row in the stage's gathered-row array
// [window | singles | groups].  The arithmetic is untouched -- the kernel still
// accumulates every row's entries in CSR order -- so the plan only changes
// where the gathered values are read from.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstdint>
#include <thread>
#include <vector>

#include "phx_kernels.cuh"

namespace phx {

namespace {

struct TileInfo {
  int32_t ng = 0;
  int32_t goff[kPlanGroups] = {0, 0, 0, 0};
  int32_t nsgl = 0;
  int32_t ne = 0;
  bool ok = true;
};

// groups and singles of one tile (deterministic: groups by count desc, then
// offset asc; singles sorted by column)
// Rows are the part's (n of them, the first one global row row0; rp points at
// the part's first row_ptr entry, ci is the whole column array); columns and
// the window are global rows of an operator of ntot rows.
void analyse_tile(int64_t n, const int64_t* rp, const int32_t* ci, int64_t row0, int64_t ntot,
                  int64_t t, TileInfo* info, std::vector<int32_t>* singles,
                  std::vector<int64_t>& scratch) {
  const int64_t base = t * kPlanT, rows = std::min<int64_t>(kPlanT, n - base);
  const int64_t gb = row0 + base;
  const int64_t wlo = std::max<int64_t>(gb - 1, 0), whi = std::min<int64_t>(gb + rows + 1, ntot);
  scratch.clear();
  for (int64_t rr = 0; rr < rows; ++rr)
    for (int64_t e = rp[base + rr]; e < rp[base + rr + 1]; ++e) {
      const int64_t col = ci[e];
      if (col >= wlo && col < whi) continue;
      scratch.push_back(col - (gb + rr));
    }
  info->ne = int32_t(rp[base + rows] - rp[base]);
  std::sort(scratch.begin(), scratch.end());
  std::vector<std::pair<int64_t, int64_t>> runs;  // (-count, offset)
  for (size_t i = 0; i < scratch.size();) {
    size_t j = i;
    while (j < scratch.size() && scratch[j] == scratch[i]) ++j;
    runs.push_back({-int64_t(j - i), scratch[i]});
    i = j;
  }
  std::sort(runs.begin(), runs.end());
  const int64_t need = std::max<int64_t>(2, rows / 4);
  info->ng = 0;
  for (const auto& rc : runs) {
    if (info->ng >= kPlanGroups || -rc.first < need) break;
    info->goff[info->ng++] = int32_t(rc.second);
  }
  // singles: distinct columns of the remaining out-of-window entries
  std::vector<int32_t> sg;
  for (int64_t rr = 0; rr < rows; ++rr)
    for (int64_t e = rp[base + rr]; e < rp[base + rr + 1]; ++e) {
      const int64_t col = ci[e];
      if (col >= wlo && col < whi) continue;
      const int64_t off = col - (gb + rr);
      bool grouped = false;
      for (int g = 0; g < info->ng; ++g) grouped = grouped || info->goff[g] == off;
      if (!grouped) sg.push_back(int32_t(col));
    }
  std::sort(sg.begin(), sg.end());
  sg.erase(std::unique(sg.begin(), sg.end()), sg.end());
  info->nsgl = int32_t(sg.size());
  info->ok = info->nsgl <= kPlanMaxSingles && info->ne <= kPlanMaxEntries;
  if (singles) *singles = std::move(sg);
}

template <class F>
void parallel_tiles(int64_t ntiles, F&& f) {
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  const int64_t nthr = std::min<int64_t>(int64_t(hw), std::max<int64_t>(1, ntiles / 4096));
  std::atomic<int64_t> next{0};
  auto work = [&] {
    std::vector<int64_t> scratch;
    for (;;) {
      const int64_t t0 = next.fetch_add(1024);
      if (t0 >= ntiles) return;
      for (int64_t t = t0; t < std::min(ntiles, t0 + 1024); ++t) f(t, scratch);
    }
  };
  std::vector<std::thread> th;
  for (int64_t i = 1; i < nthr; ++i) th.emplace_back(work);
  work();
  for (auto& x : th) x.join();
}

// Processing order of the tiles (the kernel hands out positions in this
// order; the descriptors are stored in it, d[5] = the tile).  Lattice
// operators -- offset groups +-B1 and +-B2 with T | B1 | B2 | n, e.g. a 3D
// 7-point stencil (B1 = nx, B2 = nx*ny) -- are swept in y-blocks of kYBlock
// lines: for each block, for z, for y in the block, for the x tiles.  A row
// is then gathered again (as a z-1 neighbour) 2 * kYBlock lines after its
// first use instead of two whole planes later, so the reuse fits in L2
// (C3: 3.9 MB instead of 31 MB of D per reuse window).  Other operators keep
// the natural order.
constexpr int64_t kYBlock = 32;
void tile_order(int64_t n, int64_t row0, const std::vector<TileInfo>& info, TilePlan* plan) {
  const int64_t T = kPlanT, ntiles = int64_t(info.size());
  std::vector<int32_t> order(static_cast<size_t>(ntiles));
  for (int64_t t = 0; t < ntiles; ++t) order[size_t(t)] = int32_t(t);
  // the lattice strides: the two largest |group offsets| present in at least
  // half of the tiles, as +- pairs
  std::vector<std::pair<int64_t, int64_t>> cnt;  // (|off|, tiles)
  for (const TileInfo& ti : info)
    for (int g = 0; g < ti.ng; ++g) {
      const int64_t a = std::abs(int64_t(ti.goff[g]));
      bool f = false;
      for (auto& c : cnt)
        if (c.first == a) {
          ++c.second;
          f = true;
        }
      if (!f && cnt.size() < 64) cnt.push_back({a, 1});
    }
  std::vector<int64_t> strides;
  for (const auto& c : cnt)
    if (c.second >= ntiles) strides.push_back(c.first);  // +off and -off in >= half the tiles
  std::sort(strides.begin(), strides.end());
  const char* env = std::getenv("PHX_PLAN_BLOCKED");  // developer knob (read at creation)
  if (strides.size() >= 2 && !(env && env[0] == '0')) {
    const int64_t B2 = strides.back(), B1 = strides[strides.size() - 2];
    if (B1 % T == 0 && B2 % B1 == 0 && n % B2 == 0 && row0 % B2 == 0 && B2 / B1 >= 2 * kYBlock) {
      const int64_t ny = B2 / B1, nz = n / B2, xt = B1 / T;
      size_t q = 0;
      for (int64_t yb = 0; yb < ny; yb += kYBlock)
        for (int64_t z = 0; z < nz; ++z)
          for (int64_t y = yb; y < std::min(ny, yb + kYBlock); ++y)
            for (int64_t x = 0; x < xt; ++x) order[q++] = int32_t((z * B2 + y * B1) / T + x);
      plan->blocked = true;
    }
  }
  std::vector<int32_t> desc(plan->desc.size());
  for (int64_t q = 0; q < ntiles; ++q) {
    const int32_t t = order[size_t(q)];
    std::copy(plan->desc.begin() + size_t(t) * kPlanDesc,
              plan->desc.begin() + size_t(t + 1) * kPlanDesc, desc.begin() + size_t(q) * kPlanDesc);
    desc[size_t(q) * kPlanDesc + 5] = t;
  }
  plan->desc.swap(desc);
}

}  // namespace

bool build_tile_plan(int64_t n, const int64_t* rp, const int32_t* ci, TilePlan* plan, int64_t row0,
                     int64_t ntot) {
  plan->ok = false;
  if (ntot < 0) ntot = n;
  const int64_t ntiles = (n + kPlanT - 1) / kPlanT;
  std::vector<TileInfo> info(static_cast<size_t>(ntiles));
  std::atomic<bool> ok{true};
  parallel_tiles(ntiles, [&](int64_t t, std::vector<int64_t>& scratch) {
    if (!ok.load(std::memory_order_relaxed)) return;
    analyse_tile(n, rp, ci, row0, ntot, t, &info[size_t(t)], nullptr, scratch);
    if (!info[size_t(t)].ok) ok = false;
  });
  if (!ok) return false;
  int32_t ngmax = 0, smax = 0, emax = 0;
  std::vector<int64_t> sgl_lo(size_t(ntiles) + 1, 0);
  for (int64_t t = 0; t < ntiles; ++t) {
    ngmax = std::max(ngmax, info[size_t(t)].ng);
    smax = std::max(smax, info[size_t(t)].nsgl);
    emax = std::max(emax, info[size_t(t)].ne);
    sgl_lo[size_t(t + 1)] = sgl_lo[size_t(t)] + info[size_t(t)].nsgl;
  }
  if (sgl_lo[size_t(ntiles)] >= (int64_t(1) << 31)) return false;
  const int32_t T = kPlanT;
  const int32_t gbase = (T + 2) + smax;  // first group row of a stage
  plan->rows = gbase + ngmax * T;
  plan->sgl_cap = smax;
  plan->emax = (emax + 1) / 2 * 2;
  if (plan->rows > 256) return false;  // one-byte slots
  const int64_t e0 = rp[0], nnz = rp[n] - e0;  // the part's entries (slots are part-local)
  plan->desc.assign(size_t(ntiles) * kPlanDesc, 0);
  plan->slot.assign(size_t(nnz) + 16, 0);
  plan->sgl.assign(size_t(sgl_lo[size_t(ntiles)]) + 1, 0);
  parallel_tiles(ntiles, [&](int64_t t, std::vector<int64_t>& scratch) {
    TileInfo ti;
    std::vector<int32_t> sg;
    analyse_tile(n, rp, ci, row0, ntot, t, &ti, &sg, scratch);
    const int64_t base = t * T, rows = std::min<int64_t>(T, n - base);
    const int64_t gb = row0 + base;
    const int64_t wlo = std::max<int64_t>(gb - 1, 0), whi = std::min<int64_t>(gb + rows + 1, ntot);
    int32_t* d = plan->desc.data() + size_t(t) * kPlanDesc;
    d[0] = ti.ng;
    d[1] = ti.nsgl;
    d[2] = int32_t(sgl_lo[size_t(t)]);
    d[3] = int32_t(rp[base] - e0);
    d[4] = int32_t(rp[base + rows] - e0);
    for (int g = 0; g < ti.ng; ++g) {
      const int64_t o0 = gb + ti.goff[g];
      const int64_t s0 = std::max<int64_t>(0, o0), s1 = std::min<int64_t>(ntot, o0 + rows);
      const int64_t dst = gbase + int64_t(g) * T + (s0 - o0);
      d[8 + g] = int32_t(s0);
      d[12 + g] = int32_t((s1 - s0) | (dst << 16));
    }
    std::copy(sg.begin(), sg.end(), plan->sgl.begin() + sgl_lo[size_t(t)]);
    for (int64_t rr = 0; rr < rows; ++rr)
      for (int64_t e = rp[base + rr]; e < rp[base + rr + 1]; ++e) {
        const int64_t col = ci[e];
        int64_t sl;
        if (col >= wlo && col < whi) {
          sl = col - wlo;
        } else {
          const int64_t off = col - (gb + rr);
          int g = -1;
          for (int q = 0; q < ti.ng; ++q)
            if (ti.goff[q] == off) g = q;
          if (g >= 0)
            sl = gbase + int64_t(g) * T + rr;
          else
            sl = (T + 2) + (std::lower_bound(sg.begin(), sg.end(), int32_t(col)) - sg.begin());
        }
        plan->slot[size_t(e - e0)] = uint8_t(sl);
      }
  });
  tile_order(n, row0, info, plan);
  plan->ok = true;
  return true;
}

}  // namespace phx
