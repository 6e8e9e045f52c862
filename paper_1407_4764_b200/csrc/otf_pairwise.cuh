// otf_pairwise.cuh — numpy's pairwise summation order on the device (shared by the PQ scan,
// the k-means objective and the ingest normalisation). Restated and pinned against numpy in
// oracle/otf_oracle.py::pairwise_sum_numpy_order.
#pragma once

#include "otf_common.cuh"

namespace otf {

// numpy pairwise sum (n <= 128 branch and the recursive split), values from a getter.
template <typename Get>
__device__ __forceinline__ double pairwise_block(const Get& a, int s, int n) {
  if (n < 8) {
    double res = -0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, a(s + i));
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a(s + j);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a(s + i + j));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, a(s + i));
  return res;
}
template <typename Get>
__device__ double pairwise_sum(const Get& a, int s, int n) {
  if (n <= 128) return pairwise_block(a, s, n);
  // explicit stack instead of recursion: numpy splits at n2 = (n/2) - (n/2)%8
  // and returns pairwise(left) + pairwise(right). Depth <= log2(n/128)+1.
  struct Frame { int s, n, stage; double left; };
  Frame st[24];
  int top = 0;
  st[0] = {s, n, 0, 0.0};
  double ret = 0.0;
  while (top >= 0) {
    Frame& f = st[top];
    if (f.n <= 128) { ret = pairwise_block(a, f.s, f.n); --top; continue; }
    int n2 = f.n / 2; n2 -= n2 % 8;
    if (f.stage == 0) { f.stage = 1; st[top + 1] = {f.s, n2, 0, 0.0}; ++top; continue; }
    if (f.stage == 1) { f.left = ret; f.stage = 2; st[top + 1] = {f.s + n2, f.n - n2, 0, 0.0}; ++top; continue; }
    ret = __dadd_rn(f.left, ret);
    --top;
  }
  return ret;
}

}  // namespace otf
