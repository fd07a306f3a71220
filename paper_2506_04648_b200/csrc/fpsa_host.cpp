// Host-side layout logic of the hot path: tile grid, tile permutation,
// sliding-tile window CSR, step regime, attention work list.
//
// Reference semantics followed (all under /root/reference/pkg/src/fp8sta):
//   grid.py:91-109      tile grid + indivisible-axis error text
//   grid.py:132-154     tile-major gather permutation
//   sparsity.py:43-45   window reach: back (W-1)/2, forward W/2, clipped
//   sparsity.py:63-75   allowed(u): ascending flat key-tile ids
//   schedule.py:41-50   regime thresholds floor(alpha*D), boundary -> earlier
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/fpsa.h"
#include "fpsa_internal.h"

namespace {
thread_local std::string g_last_error;
}

namespace fpsa {
int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}
void clear_error() { g_last_error.clear(); }
}  // namespace fpsa

using fpsa::fail;

extern "C" const char* fpsa_last_error(void) { return g_last_error.c_str(); }

extern "C" int fpsa_version(void) { return 1 * 10000 + 0 * 100 + 0; }

static int check_dims(const char* what, fpsa_dims3 d) {
  const int32_t v[3] = {d.t, d.h, d.w};
  const char* names[3] = {"t", "h", "w"};
  for (int i = 0; i < 3; ++i)
    if (v[i] < 1)
      return fail(FPSA_EINVAL, std::string(what) + "." + names[i] + " must be >= 1, got " + std::to_string(v[i]));
  return FPSA_OK;
}

extern "C" int fpsa_tile_grid(fpsa_dims3 grid, fpsa_dims3 tile, fpsa_dims3* tile_dims) {
  fpsa::clear_error();
  if (int s = check_dims("grid", grid)) return s;
  if (int s = check_dims("tile", tile)) return s;
  const int32_t g[3] = {grid.t, grid.h, grid.w};
  const int32_t s[3] = {tile.t, tile.h, tile.w};
  const char axes[3] = {'t', 'h', 'w'};
  int32_t out[3];
  for (int i = 0; i < 3; ++i) {
    if (g[i] % s[i] != 0) {
      char buf[160];
      snprintf(buf, sizeof buf, "indivisible grid: axis %c has %d tokens, not divisible by tile extent %d", axes[i],
               g[i], s[i]);
      return fail(FPSA_EINDIVISIBLE, buf);
    }
    out[i] = g[i] / s[i];
  }
  if (tile_dims) *tile_dims = fpsa_dims3{out[0], out[1], out[2]};
  return FPSA_OK;
}

extern "C" int fpsa_tile_perm(fpsa_dims3 grid, fpsa_dims3 tile, int64_t* perm) {
  fpsa_dims3 td;
  if (int s = fpsa_tile_grid(grid, tile, &td)) return s;
  if (!perm) return fail(FPSA_EINVAL, "perm is NULL");
  const int64_t tv = (int64_t)tile.t * tile.h * tile.w;
  int64_t pos = 0;
  // Walk destinations in order: tiles row-major, tokens row-major inside.
  for (int32_t ut = 0; ut < td.t; ++ut)
    for (int32_t uh = 0; uh < td.h; ++uh)
      for (int32_t uw = 0; uw < td.w; ++uw)
        for (int32_t lt = 0; lt < tile.t; ++lt)
          for (int32_t lh = 0; lh < tile.h; ++lh) {
            const int64_t t = (int64_t)ut * tile.t + lt, h = (int64_t)uh * tile.h + lh;
            const int64_t row0 = (t * grid.h + h) * grid.w + (int64_t)uw * tile.w;
            for (int32_t lw = 0; lw < tile.w; ++lw) perm[pos++] = row0 + lw;
          }
  (void)tv;
  return FPSA_OK;
}

namespace {
inline void axis_range(int32_t x, int32_t dim, int32_t extent, int32_t* lo, int32_t* hi) {
  const int32_t back = (extent - 1) / 2, fwd = extent / 2;
  *lo = std::max(0, x - back);
  *hi = std::min(dim - 1, x + fwd);
}
}  // namespace

extern "C" int fpsa_window_nnz(fpsa_dims3 td, fpsa_dims3 win, int64_t* nnz) {
  fpsa::clear_error();
  if (td.t < 1 || td.h < 1 || td.w < 1) {
    char buf[128];
    snprintf(buf, sizeof buf, "tile grid dims must be >= 1, got (%d, %d, %d)", td.t, td.h, td.w);
    return fail(FPSA_EINVAL, buf);
  }
  if (win.t < 1) return fail(FPSA_EINVAL, "WindowSpec.win_t must be >= 1, got " + std::to_string(win.t));
  if (win.h < 1) return fail(FPSA_EINVAL, "WindowSpec.win_h must be >= 1, got " + std::to_string(win.h));
  if (win.w < 1) return fail(FPSA_EINVAL, "WindowSpec.win_w must be >= 1, got " + std::to_string(win.w));
  // The admissible set factorises per axis, so the total is a product of sums.
  const int32_t dims[3] = {td.t, td.h, td.w}, ext[3] = {win.t, win.h, win.w};
  int64_t total = 1;
  for (int a = 0; a < 3; ++a) {
    int64_t s = 0;
    for (int32_t x = 0; x < dims[a]; ++x) {
      int32_t lo, hi;
      axis_range(x, dims[a], ext[a], &lo, &hi);
      s += hi - lo + 1;
    }
    total *= s;
  }
  if (nnz) *nnz = total;
  return FPSA_OK;
}

extern "C" int fpsa_window_csr(fpsa_dims3 td, fpsa_dims3 win, int32_t* offs, int32_t* ids, int64_t cap,
                               int64_t* nnz) {
  int64_t total = 0;
  if (int s = fpsa_window_nnz(td, win, &total)) return s;
  if (nnz) *nnz = total;
  if (!offs || !ids) return fail(FPSA_EINVAL, "offs/ids is NULL");
  if (cap < total) return fail(FPSA_ECAPACITY, "ids capacity " + std::to_string(cap) + " < nnz " + std::to_string(total));
  int64_t pos = 0;
  int32_t u = 0;
  offs[0] = 0;
  for (int32_t ut = 0; ut < td.t; ++ut) {
    int32_t t0, t1;
    axis_range(ut, td.t, win.t, &t0, &t1);
    for (int32_t uh = 0; uh < td.h; ++uh) {
      int32_t h0, h1;
      axis_range(uh, td.h, win.h, &h0, &h1);
      for (int32_t uw = 0; uw < td.w; ++uw) {
        int32_t w0, w1;
        axis_range(uw, td.w, win.w, &w0, &w1);
        for (int32_t vt = t0; vt <= t1; ++vt)
          for (int32_t vh = h0; vh <= h1; ++vh) {
            const int32_t base = (vt * td.h + vh) * td.w;
            for (int32_t vw = w0; vw <= w1; ++vw) ids[pos++] = base + vw;
          }
        offs[++u] = (int32_t)pos;
      }
    }
  }
  return FPSA_OK;
}

extern "C" int fpsa_regime_of(int32_t t, int32_t total, double alpha1, double alpha2, int32_t* regime) {
  fpsa::clear_error();
  if (t < 1 || t > total)
    return fail(FPSA_EINVAL, "step " + std::to_string(t) + " out of range [1, " + std::to_string(total) + "]");
  const int64_t t1 = (int64_t)std::floor(alpha1 * total), t2 = (int64_t)std::floor(alpha2 * total);
  *regime = t <= t1 ? 0 : (t <= t2 ? 1 : 2);
  return FPSA_OK;
}

extern "C" int fpsa_attn_worklist(int32_t heads, fpsa_dims3 td, int32_t tile_volume, const int32_t* offs,
                                  int32_t* items, int64_t cap, int64_t* n_items) {
  fpsa::clear_error();
  if (heads < 1 || tile_volume < 1 || !offs) return fail(FPSA_EINVAL, "bad worklist arguments");
  const int32_t M = td.t * td.h * td.w;
  const int32_t nqb = (tile_volume + 127) / 128;  // 128-row query blocks per tile
  // Longest-processing-time first inside each head; heads in order so that the
  // K/V codes of the heads in flight stay L2 resident.
  std::vector<int32_t> order(M);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t a, int32_t b) { return offs[a + 1] - offs[a] > offs[b + 1] - offs[b]; });
  const int64_t total = (int64_t)heads * M * nqb;
  if (n_items) *n_items = total;
  if (!items) return FPSA_OK;
  if (cap < total) return fail(FPSA_ECAPACITY, "work list capacity too small");
  int64_t pos = 0;
  for (int32_t h = 0; h < heads; ++h)
    for (int32_t i = 0; i < M; ++i)
      for (int32_t qb = 0; qb < nqb; ++qb) {
        items[3 * pos + 0] = h;
        items[3 * pos + 1] = order[i];
        items[3 * pos + 2] = qb;
        ++pos;
      }
  return FPSA_OK;
}
