// Host-side (CPU) mesh topology kernels of the table builder, native for
// large meshes.  Both reproduce the numpy builder exactly:
//   mhdg_pair_sides   : skeleton pairing of macro sides by their canonical
//                       quantised vertex keys (reference mesh.py:226-299;
//                       our mesh.skeleton_arrays)
//   mhdg_match_points : trace-node matching of a face's neighbour side to
//                       the owner's node order (reference assembly.py:
//                       299-322, nearest point; our tables.HDGTables._trace)
// Integer outputs are bit-identical to the numpy implementation (same
// lexicographic key order, same first-minimum argmin over the same
// floating-point distances).
#pragma once
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

namespace mhdg_host {

// partner[s] = the other side with the same key, -1 if unique; returns the
// number of key groups with more than two sides (a topology error)
inline int64_t pair_sides(int64_t n, int w, const int64_t* keys, int64_t* partner) {
  std::vector<int64_t> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  auto less = [&](int64_t a, int64_t b) {
    const int64_t* ka = keys + a * w;
    const int64_t* kb = keys + b * w;
    for (int c = 0; c < w; ++c)
      if (ka[c] != kb[c]) return ka[c] < kb[c];
    return a < b;
  };
  std::sort(idx.begin(), idx.end(), less);
  auto same = [&](int64_t a, int64_t b) {
    const int64_t* ka = keys + a * w;
    const int64_t* kb = keys + b * w;
    for (int c = 0; c < w; ++c)
      if (ka[c] != kb[c]) return false;
    return true;
  };
  int64_t bad = 0;
  for (int64_t s = 0; s < n; ++s) partner[s] = -1;
  for (int64_t i = 0; i < n;) {
    int64_t j = i + 1;
    while (j < n && same(idx[i], idx[j])) ++j;
    if (j - i == 2) {
      partner[idx[i]] = idx[i + 1];
      partner[idx[i + 1]] = idx[i];
    } else if (j - i > 2) {
      ++bad;
    }
    i = j;
  }
  return bad;
}

// match[f][a] = argmin_b |pb[f][a] - po[f][b]| (first minimum), per face;
// returns the largest best distance and flags duplicate matches (-1.0)
inline double match_points(int64_t nf, int nt, int d, const double* pb, const double* po, int64_t* match) {
  double worst = 0.0;
  std::vector<int64_t> seen(nt);
  for (int64_t f = 0; f < nf; ++f) {
    const double* b = pb + f * nt * d;
    const double* o = po + f * nt * d;
    for (int a = 0; a < nt; ++a) {
      double best = INFINITY;
      int bi = 0;
      for (int c = 0; c < nt; ++c) {
        double s = 0.0;
        for (int k = 0; k < d; ++k) {
          const double df = b[a * d + k] - o[c * d + k];
          s += df * df;
        }
        const double dist = std::sqrt(s);
        if (dist < best) {
          best = dist;
          bi = c;
        }
      }
      match[f * nt + a] = bi;
      worst = std::max(worst, best);
    }
    for (int a = 0; a < nt; ++a) seen[a] = 0;
    for (int a = 0; a < nt; ++a)
      if (seen[match[f * nt + a]]++) return -1.0;
  }
  return worst;
}

// Neighbour-side trace nodes built on the fly and matched to the owner's
// node order (tables.HDGTables._trace): for face f, node a of the
// neighbour's local face nfl: x = origin[ne] + J[ne] fun[nfl][a] - shift[f]
// (the points only decide an argmin between well separated nodes; their
// last bits do not matter), then the first-minimum match against po.
inline double match_faces(int64_t nf, int nt, int d, const double* fun, const int64_t* ne, const int64_t* nfl,
                          const double* origins, const double* jac, const double* shift, const double* po,
                          int64_t* match) {
  std::vector<double> pb((size_t)nt * d);
  double worst = 0.0;
  for (int64_t f = 0; f < nf; ++f) {
    const double* org = origins + ne[f] * d;
    const double* J = jac + ne[f] * d * d;
    const double* fu = fun + nfl[f] * nt * d;
    for (int a = 0; a < nt; ++a)
      for (int c = 0; c < d; ++c) {
        double x = 0.0;
        for (int b = 0; b < d; ++b) x += fu[a * d + b] * J[c * d + b];
        pb[a * d + c] = (org[c] + x) - shift[f * d + c];
      }
    const double w = match_points(1, nt, d, pb.data(), po + f * nt * d, match + f * nt);
    if (w < 0) return -1.0;
    worst = std::max(worst, w);
  }
  return worst;
}

// Canonical side keys (mesh.skeleton_arrays, reference mesh.py:226-299):
// sv (S, d, d) side vertex coordinates; vertices on a periodic max plane are
// wrapped by -extent, quantised to round(x / quantum) (round half to even,
// numpy's np.round), and each side's d vertex rows sorted lexicographically.
inline void side_keys(int64_t n_sides, int d, const double* sv, const double* box_hi, const double* extent,
                      const int* periodic, double quantum, int64_t* keys) {
  for (int64_t sdx = 0; sdx < n_sides; ++sdx) {
    const double* v = sv + sdx * d * d;
    int64_t* k = keys + sdx * d * d;
    for (int a = 0; a < d; ++a) {
      bool on_max = periodic[a] != 0;
      for (int r = 0; r < d && on_max; ++r) on_max = std::fabs(v[r * d + a] - box_hi[a]) < quantum;
      for (int r = 0; r < d; ++r) {
        const double x = on_max ? v[r * d + a] - extent[a] : v[r * d + a];
        k[r * d + a] = (int64_t)std::nearbyint(x / quantum);
      }
    }
    // insertion sort of the d rows (stable, lexicographic)
    for (int i = 1; i < d; ++i)
      for (int j = i; j > 0; --j) {
        int64_t* a0 = k + (j - 1) * d;
        int64_t* a1 = k + j * d;
        int c = 0;
        while (c < d && a0[c] == a1[c]) ++c;
        if (c < d && a0[c] > a1[c]) {
          for (int e = 0; e < d; ++e) std::swap(a0[e], a1[e]);
        } else {
          break;
        }
      }
  }
}

// Periodic shift and vertex permutation of paired faces (same float
// operations as the numpy builder: centroid = ((v0 + v1) + v2) / d,
// shift = round(delta / extent) * extent, distance = sqrt of the ordered
// sum of squares, first-minimum argmin).  Returns the largest matched
// distance, or -1 for a degenerate matching.
inline double face_shift_perm(int64_t nf, int d, const double* va, const double* vb, const double* extent,
                              double* shift, int64_t* perm) {
  double worst = 0.0;
  for (int64_t f = 0; f < nf; ++f) {
    const double* a = va + f * d * d;
    const double* b = vb + f * d * d;
    double* sh = shift + f * d;
    for (int c = 0; c < d; ++c) {
      double sa = a[c], sb = b[c];
      for (int r = 1; r < d; ++r) {
        sa += a[r * d + c];
        sb += b[r * d + c];
      }
      const double delta = sb / d - sa / d;
      sh[c] = std::nearbyint(delta / extent[c]) * extent[c];
    }
    int64_t* pm = perm + f * d;
    for (int i = 0; i < d; ++i) {
      double best = 0.0;
      int bj = -1;
      for (int j = 0; j < d; ++j) {
        double acc = 0.0;
        for (int c = 0; c < d; ++c) {
          const double t = (b[j * d + c] - sh[c]) - a[i * d + c];
          acc += t * t;
        }
        const double dist = std::sqrt(acc);
        if (bj < 0 || dist < best) {
          best = dist;
          bj = j;
        }
      }
      pm[i] = bj;
      worst = std::max(worst, best);
    }
    for (int i = 0; i < d; ++i)
      for (int j = i + 1; j < d; ++j)
        if (pm[i] == pm[j]) return -1.0;
  }
  return worst;
}

}  // namespace mhdg_host
