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

}  // namespace mhdg_host
