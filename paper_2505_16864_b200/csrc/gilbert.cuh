// Closed-form position of a cell on the generalized-Hilbert ("gilbert") plane curve
// and on the slab-paired 3D curve of the reference (sfc.py:98-210).
//
// Instead of emitting the whole curve recursively (the reference walks the recursion
// and appends cells, sfc.py:116-157), every cell descends the same split tree and
// adds the sizes of the sub-rectangles that precede the one containing it: depth is
// O(log max(a,b)), so one thread per cell suffices.  Host+device so the CPU tests can
// check the descent exhaustively against the reference order without a GPU.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define TCB_HD __host__ __device__ __forceinline__
#else
#define TCB_HD inline
#endif

namespace tcb {

TCB_HD int isgn(int v) { return (v > 0) - (v < 0); }
TCB_HD int iabs(int v) { return v < 0 ? -v : v; }
// Python floor division by 2 (sfc.py:133-134 relies on it for negative vectors).
TCB_HD int floordiv2(int a) { return a >= 0 ? a / 2 : -((-a + 1) / 2); }

// Rectangle of the split tree: origin (x,y), major vector a, minor vector b.
struct GRect {
  int x, y, ax, ay, bx, by;
};

TCB_HD int64_t grect_cells(const GRect& r) {
  return (int64_t)iabs(r.ax + r.ay) * (int64_t)iabs(r.bx + r.by);
}

// a and b are always axis-aligned and orthogonal, so (i, j) decomposes the offset.
TCB_HD bool grect_has(const GRect& r, int tx, int ty) {
  int rx = tx - r.x, ry = ty - r.y;
  int i = rx * isgn(r.ax) + ry * isgn(r.ay);
  int j = rx * isgn(r.bx) + ry * isgn(r.by);
  return i >= 0 && j >= 0 && i < iabs(r.ax + r.ay) && j < iabs(r.bx + r.by);
}

// Curve position of plane cell (tx, ty) in the a x b gilbert order (sfc.py:98-109).
TCB_HD int64_t gilbert_index(int a, int b, int tx, int ty) {
  GRect r = (a >= b) ? GRect{0, 0, a, 0, 0, b} : GRect{0, 0, 0, b, a, 0};
  int64_t off = 0;
  for (;;) {
    const int w = iabs(r.ax + r.ay), h = iabs(r.bx + r.by);
    const int dax = isgn(r.ax), day = isgn(r.ay), dbx = isgn(r.bx), dby = isgn(r.by);
    const int rx = tx - r.x, ry = ty - r.y;
    if (h == 1) return off + rx * dax + ry * day;   // straight run along a (sfc.py:123-127)
    if (w == 1) return off + rx * dbx + ry * dby;   // straight run along b (sfc.py:128-132)
    int ax2 = floordiv2(r.ax), ay2 = floordiv2(r.ay);
    int bx2 = floordiv2(r.bx), by2 = floordiv2(r.by);
    const int w2 = iabs(ax2 + ay2), h2 = iabs(bx2 + by2);
    if (2 * w > 3 * h) {                            // two-way split (sfc.py:138-143)
      if ((w2 & 1) && w > 2) { ax2 += dax; ay2 += day; }
      GRect c0{r.x, r.y, ax2, ay2, r.bx, r.by};
      if (grect_has(c0, tx, ty)) { r = c0; continue; }
      off += grect_cells(c0);
      r = GRect{r.x + ax2, r.y + ay2, r.ax - ax2, r.ay - ay2, r.bx, r.by};
    } else {                                        // three-way split (sfc.py:144-157)
      if ((h2 & 1) && h > 2) { bx2 += dbx; by2 += dby; }
      GRect c0{r.x, r.y, bx2, by2, ax2, ay2};
      if (grect_has(c0, tx, ty)) { r = c0; continue; }
      off += grect_cells(c0);
      GRect c1{r.x + bx2, r.y + by2, r.ax, r.ay, r.bx - bx2, r.by - by2};
      if (grect_has(c1, tx, ty)) { r = c1; continue; }
      off += grect_cells(c1);
      r = GRect{r.x + (r.ax - dax) + (bx2 - dbx), r.y + (r.ay - day) + (by2 - dby),
                -bx2, -by2, -(r.ax - ax2), -(r.ay - ay2)};
    }
  }
}

// Geometry of the 3D curve: slab axis = argmin(t,h,w) (ties -> lowest axis), plane
// axes p1 < p2 the other two (sfc.py:163-165).
struct CurveGeom {
  int dims[3];
  int s_ax, p1, p2;
  int64_t n_plane;
};

TCB_HD CurveGeom curve_geom(int t, int h, int w) {
  CurveGeom g;
  g.dims[0] = t; g.dims[1] = h; g.dims[2] = w;
  int s = 0;
  if (g.dims[1] < g.dims[s]) s = 1;
  if (g.dims[2] < g.dims[s]) s = 2;
  g.s_ax = s;
  g.p1 = (s == 0) ? 1 : 0;
  g.p2 = (s == 2) ? 1 : 2;
  g.n_plane = (int64_t)g.dims[g.p1] * g.dims[g.p2];
  return g;
}

// Curve position of row-major cell c (sfc.py:166-195 in closed form): slices are
// consumed in pairs (lo=2q, hi=2q+1) walking the plane forward for even q and
// reversed for odd q, zig-zagging lo/hi per plane cell with the last cell forced
// to exit on hi; a trailing odd slice is walked once.
TCB_HD int64_t curve_position(const CurveGeom& g, int64_t c) {
  const int64_t hw = (int64_t)g.dims[1] * g.dims[2];
  int coord[3];
  coord[0] = (int)(c / hw);
  int64_t rem = c - (int64_t)coord[0] * hw;
  coord[1] = (int)(rem / g.dims[2]);
  coord[2] = (int)(rem - (int64_t)coord[1] * g.dims[2]);
  const int s = coord[g.s_ax];
  const int64_t i_fwd = gilbert_index(g.dims[g.p1], g.dims[g.p2], coord[g.p1], coord[g.p2]);
  const int q = s >> 1;
  const int64_t i = (q & 1) ? (g.n_plane - 1 - i_fwd) : i_fwd;
  const int64_t base = 2 * g.n_plane * (int64_t)q;
  if (2 * q + 1 < g.dims[g.s_ax]) {
    const bool lo = (s == 2 * q);
    const bool lo_first = ((i & 1) == 0) || (i == g.n_plane - 1);
    return base + 2 * i + ((lo == lo_first) ? 0 : 1);
  }
  return base + i;
}

}  // namespace tcb
