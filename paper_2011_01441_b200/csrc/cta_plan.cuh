// CTA-level plans shared by host and device: the PACO cuboid plan
// (plan_piece, PACO_MM_PACO_PLAN) and the default tile grid (plan_grid_piece).
//
// The recursion is mm_one_piece_partition's (matmul.py:250-300): the worker
// list [lo, hi) splits floor(cnt/2) : ceil(cnt/2); the cut axis is the longest
// axis of an evenly halved virtual cuboid (ties n -> m -> k); the real length
// is split in the worker ratio.  Two changes are forced by tile quantisation
// (C tiles of bm x bn, k quanta of kq elements): the cut lands on the NEAREST
// unit, and when that cut on the virtual axis would miss the worker ratio by
// more than 1%, the axis with the smallest miss is cut instead (k is the fine
// axis).  paco_plan_cta() runs it on the host; simt_mm_kernel runs the same
// descent per CTA (O(log p) steps) so a plan needs no table.
#pragma once
#include <cstdint>

namespace paco {

struct UnitBox {
  int64_t o[3];  // offsets in units (C tiles along n, m; k quanta along k)
  int64_t e[3];  // extents in units
};

struct PlanStep {
  int axis;      // -1: infeasible (an extent of 1 had to be cut)
  int64_t left;  // units kept by the lower worker half
};

__host__ __device__ inline int plan_virtual_axis(const double v[3]) {
  if (v[0] >= v[1] && v[0] >= v[2]) return 0;
  return v[1] >= v[2] ? 1 : 2;
}

__host__ __device__ inline int64_t plan_cut_at(int64_t len, int h, int cnt) {
  int64_t left = (2 * len * h + cnt) / (2 * cnt);  // nearest unit to len*h/cnt
  if (left < 1) left = 1;
  if (left > len - 1) left = len - 1;
  return left;
}

__host__ __device__ inline double plan_miss(int64_t len, int h, int cnt) {
  if (len < 2) return 1e30;
  const double frac = double(h) / double(cnt);
  const double got = double(plan_cut_at(len, h, cnt)) / double(len);
  const double d = got > frac ? got - frac : frac - got;
  return d / frac;
}

// One split of box `b` shared by `cnt` workers (cnt >= 2).
__host__ __device__ inline PlanStep plan_step(const UnitBox& b, int cnt, const double v[3]) {
  const int h = cnt / 2;
  int axis = plan_virtual_axis(v);
  if (plan_miss(b.e[axis], h, cnt) > 0.01) {
    int best = axis;
    for (int ax = 0; ax < 3; ++ax)
      if (plan_miss(b.e[ax], h, cnt) < plan_miss(b.e[best], h, cnt)) best = ax;
    axis = best;
  }
  if (b.e[axis] < 2) return PlanStep{-1, 0};
  return PlanStep{axis, plan_cut_at(b.e[axis], h, cnt)};
}

__host__ __device__ inline UnitBox plan_root(int64_t n, int64_t m, int64_t k, int bm, int bn, int kq) {
  UnitBox b;
  b.o[0] = b.o[1] = b.o[2] = 0;
  b.e[0] = (n + bm - 1) / bm;
  b.e[1] = (m + bn - 1) / bn;
  b.e[2] = (k + kq - 1) / kq;
  return b;
}

// Piece of worker `idx` among p; false if the plan is infeasible on its path.
//
// kw scales the virtual k length: 1 is the reference's rule; kw < 1 makes the
// descent cut the C tile grid before k (a k cut costs the piece a fold of its
// C block and splits each tile's k loop into more, shorter visits).
__host__ __device__ inline bool plan_piece(int64_t n, int64_t m, int64_t k, int bm, int bn, int kq,
                                           int p, int idx, UnitBox& out, double kw = 1.0) {
  UnitBox b = plan_root(n, m, k, bm, bn, kq);
  double v[3] = {double(n), double(m), double(k) * kw};
  int lo = 0, hi = p;
  while (hi - lo > 1) {
    const int cnt = hi - lo, h = cnt / 2;
    const PlanStep s = plan_step(b, cnt, v);
    if (s.axis < 0) return false;
    if (idx < lo + h) {
      b.e[s.axis] = s.left;
      hi = lo + h;
    } else {
      b.o[s.axis] += s.left;
      b.e[s.axis] -= s.left;
      lo = lo + h;
    }
    v[s.axis] /= 2;
  }
  out = b;
  return true;
}

// Tile-grid plan: piece idx = (C tile idx / s, k part idx % s); the k units
// split as evenly as possible.  C tiles are numbered in row-block bands of
// kGridBand (inside a band column by column), so the tiles in flight share a
// few A row blocks and B column blocks in L2.
//
// Tail split (tail > 1, s == 1): the first `head` tiles are whole pieces and
// the remaining tiles -- the partial last SM-wave -- are each split into
// `tail` k parts, so the last wave's work spreads over every SM instead of
// leaving (148 - remainder) SMs idle for a whole tile.
constexpr int64_t kGridBand = 8;

__host__ __device__ inline void plan_grid_piece(int64_t n, int64_t m, int64_t k, int bm, int bn, int kq,
                                                int s, int idx, UnitBox& out, int tail = 0, int64_t head = 0) {
  const UnitBox r = plan_root(n, m, k, bm, bn, kq);
  int64_t tile, part, parts;
  if (tail > 1 && idx >= head) {
    tile = head + (idx - head) / tail;
    part = (idx - head) % tail;
    parts = tail;
  } else {
    tile = idx / s;
    part = idx % s;
    parts = s;
  }
  const int64_t band = tile / (kGridBand * r.e[1]), r0 = band * kGridBand;
  const int64_t rows = r.e[0] - r0 < kGridBand ? r.e[0] - r0 : kGridBand;
  const int64_t v = tile - r0 * r.e[1];
  out.o[0] = r0 + v % rows;
  out.o[1] = v / rows;
  out.e[0] = out.e[1] = 1;
  out.o[2] = part * r.e[2] / parts;
  out.e[2] = (part + 1) * r.e[2] / parts - out.o[2];
}

}  // namespace paco
