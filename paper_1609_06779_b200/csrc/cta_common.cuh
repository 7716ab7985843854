// CTA-per-chain building blocks: the chain's links are spread over the
// threads of one CTA (thread t owns links [t*LPT, (t+1)*LPT)), per-link data
// lives in a field-major workspace ws[field * n + link] (shared memory when it
// fits, otherwise an L2-resident global slot), and chain recursions become
// CTA-wide scans.
//
// Scan = the paper's building block 1 (reference: scan_inclusive,
// proj/core/include/pardyn/scan.hpp:32-65): log-depth combine over warp
// shuffles plus one cross-warp level through shared memory.
//
// Inverse dynamics (reference: inverse_dynamics.cpp:27-164) is evaluated in
// base coordinates: with X_i = rel_i * ... * rel_0 (an SE(3) prefix product),
// every bi-diagonal recurrence of the reference,
//   V_i = Ad(rel_i) V_{i-1} + s_i      (lower, :27-51,  :53-84)
//   F_i = Ad(rel_{i+1})^T F_{i+1} + f_i (upper, :86-120),
// becomes V_i = Ad(X_i) * prefix_sum_k(Ad(X_k)^{-1} s_k) and
// F_i = Ad(X_i)^{-T} * suffix_sum_k(Ad(X_k)^T f_k): one structured SE(3)
// scan plus cheap 6-vector sums instead of three dense 6x6 affine scans; the
// velocity and bias-acceleration sums share one scan (PairOp).
#pragma once

#include "pd_batch.cuh"

namespace pd {

constexpr int kMaxWarps = 32;

// The threads a CTA-per-chain stage runs on: the whole CTA (default), or a
// warp-aligned range of it with its own named barrier (warp-specialised
// kernels run two stages on two thread groups at once).
struct CtaGroup {
  __device__ __forceinline__ int tid() const { return threadIdx.x; }
  __device__ __forceinline__ void sync() const { __syncthreads(); }
};
struct NamedGroup {
  int first;  // first thread (multiple of 32)
  int count;  // threads (multiple of 32)
  int bar;    // named barrier id (1..15; 0 is __syncthreads)
  __device__ __forceinline__ int tid() const { return (int)threadIdx.x - first; }
  __device__ __forceinline__ void sync() const {
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(count) : "memory");
  }
};

// Scratch for the cross-warp level of a scan (K <= 12 doubles per warp).
struct ScanSmem {
  double tot[kMaxWarps][12];
};

template <int K>
struct Arr {
  double v[K];
};

struct AddOp {
  template <int K>
  __device__ __forceinline__ Arr<K> operator()(const Arr<K>& earlier, const Arr<K>& later) const {
    Arr<K> o;
#pragma unroll
    for (int k = 0; k < K; ++k) o.v[k] = earlier.v[k] + later.v[k];
    return o;
  }
  template <int K>
  __device__ __forceinline__ Arr<K> identity() const {
    Arr<K> o;
#pragma unroll
    for (int k = 0; k < K; ++k) o.v[k] = 0.0;
    return o;
  }
};

// (V0, A0) pairs: V0 = sum of base-frame rate twists s_k, A0 = sum over
// j <= k of ad_{s_j}(s_k) -- the base-frame velocity and bias acceleration of
// inverse_dynamics.cpp:27-84 in ONE scan. Over a segment split into an earlier
// part E and a later part L, bilinearity of ad gives
// A(E+L) = A(E) + A(L) + ad_{V(E)}(V(L)) (the j = k terms vanish: ad_s s = 0).
struct PairOp {
  __device__ __forceinline__ Arr<12> operator()(const Arr<12>& earlier, const Arr<12>& later) const {
    const Sv ve = {mk(earlier.v[0], earlier.v[1], earlier.v[2]), mk(earlier.v[3], earlier.v[4], earlier.v[5])};
    const Sv vl = {mk(later.v[0], later.v[1], later.v[2]), mk(later.v[3], later.v[4], later.v[5])};
    const Sv cross_term = adv_apply(ve, vl);
    const double ct[6] = {cross_term.a.x, cross_term.a.y, cross_term.a.z, cross_term.l.x, cross_term.l.y,
                          cross_term.l.z};
    Arr<12> o;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      o.v[k] = earlier.v[k] + later.v[k];
      o.v[6 + k] = earlier.v[6 + k] + later.v[6 + k] + ct[k];
    }
    return o;
  }
  template <int K>
  __device__ __forceinline__ Arr<K> identity() const {
    Arr<K> o;
#pragma unroll
    for (int k = 0; k < K; ++k) o.v[k] = 0.0;
    return o;
  }
};

// SE(3) as Arr<12> = (R row-major, p). combine(earlier, later) = later * earlier,
// i.e. the later step multiplies from the left (scan.hpp:73-96).
__device__ __forceinline__ SE3d arr_to_se3(const Arr<12>& a) {
  SE3d T;
#pragma unroll
  for (int k = 0; k < 9; ++k) T.R.m[k] = a.v[k];
  T.p = mk(a.v[9], a.v[10], a.v[11]);
  return T;
}
__device__ __forceinline__ Arr<12> se3_to_arr(const SE3d& T) {
  Arr<12> a;
#pragma unroll
  for (int k = 0; k < 9; ++k) a.v[k] = T.R.m[k];
  a.v[9] = T.p.x;
  a.v[10] = T.p.y;
  a.v[11] = T.p.z;
  return a;
}
struct ComposeOp {
  __device__ __forceinline__ Arr<12> operator()(const Arr<12>& earlier, const Arr<12>& later) const {
    return se3_to_arr(compose(arr_to_se3(later), arr_to_se3(earlier)));
  }
  template <int K>
  __device__ __forceinline__ Arr<K> identity() const {
    Arr<K> o;
#pragma unroll
    for (int k = 0; k < K; ++k) o.v[k] = (k == 0 || k == 4 || k == 8) ? 1.0 : 0.0;
    return o;
  }
};

template <int K>
__device__ __forceinline__ Arr<K> shfl_up(const Arr<K>& x, int d) {
  Arr<K> o;
#pragma unroll
  for (int k = 0; k < K; ++k) o.v[k] = __shfl_up_sync(0xffffffffu, x.v[k], d);
  return o;
}
template <int K>
__device__ __forceinline__ Arr<K> shfl_down(const Arr<K>& x, int d) {
  Arr<K> o;
#pragma unroll
  for (int k = 0; k < K; ++k) o.v[k] = __shfl_down_sync(0xffffffffu, x.v[k], d);
  return o;
}
template <int K>
__device__ __forceinline__ Arr<K> shfl_idx(const Arr<K>& x, int src) {
  Arr<K> o;
#pragma unroll
  for (int k = 0; k < K; ++k) o.v[k] = __shfl_sync(0xffffffffu, x.v[k], src);
  return o;
}

// Exclusive scan of one element per thread across the CTA (thread order, or
// reversed thread order for REVERSE) over the first `nact` threads (the ones
// holding links; the rest hold identity and get unspecified results). Returns
// the combination of all earlier threads' elements (identity for the first).
// Runs only the combine rounds that can combine data: ceil_log2(min(32, nact))
// shuffle rounds plus ceil_log2(ceil(nact / 32)) cross-warp rounds, i.e.
// exactly ceil_log2(nact) Hillis-Steele rounds like scan.hpp:46-61 (the
// rounds ExecTrace reports, cta_scan_rounds). Contains three __syncthreads
// unless one warp holds every link (then none).
template <int K, bool REVERSE, class Op, class G = CtaGroup>
__device__ Arr<K> block_exclusive(const Arr<K>& x, Op op, ScanSmem& sm, int nact, const G& grp = G{}) {
  const int lane = grp.tid() & 31, warp = grp.tid() >> 5;
  const int span = nact < 32 ? nact : 32;    // lanes of a warp that can hold data
  const int nwa = (nact + 31) >> 5;          // warps holding data
  // warp inclusive scan in (reversed) lane order
  Arr<K> inc = x;
  for (int d = 1; d < span; d <<= 1) {
    const Arr<K> y = REVERSE ? shfl_down(inc, d) : shfl_up(inc, d);
    const bool take = REVERSE ? (lane + d < 32) : (lane >= d);
    if (take) inc = op(y, inc);
  }
  Arr<K> exc = REVERSE ? shfl_down(inc, 1) : shfl_up(inc, 1);
  const bool first_in_warp = REVERSE ? (lane == 31) : (lane == 0);
  if (first_in_warp) exc = op.template identity<K>();
  if (nwa == 1) return exc;  // one warp holds every link: no cross-warp level
  const int last_lane = REVERSE ? 0 : 31;
  if (lane == last_lane && warp < nwa) {
#pragma unroll
    for (int k = 0; k < K; ++k) sm.tot[warp][k] = inc.v[k];
  }
  grp.sync();
  if (warp == 0) {
    // scan of warp totals in (reversed) warp order; lane w holds warp w
    Arr<K> t;
    const bool valid = lane < nwa;
#pragma unroll
    for (int k = 0; k < K; ++k) t.v[k] = valid ? sm.tot[lane][k] : op.template identity<K>().v[k];
    Arr<K> ti = t;
    for (int d = 1; d < nwa; d <<= 1) {
      const Arr<K> y = REVERSE ? shfl_down(ti, d) : shfl_up(ti, d);
      const bool take = REVERSE ? (lane + d < nwa) : (lane >= d);
      if (take && valid) ti = op(y, ti);
    }
    Arr<K> te = REVERSE ? shfl_down(ti, 1) : shfl_up(ti, 1);
    const bool first_w = REVERSE ? (lane == nwa - 1) : (lane == 0);
    if (first_w) te = op.template identity<K>();
    __syncwarp();
    if (valid) {
#pragma unroll
      for (int k = 0; k < K; ++k) sm.tot[lane][k] = te.v[k];
    }
  }
  grp.sync();
  Arr<K> wp = op.template identity<K>();
  if (warp < nwa) {
#pragma unroll
    for (int k = 0; k < K; ++k) wp.v[k] = sm.tot[warp][k];
  }
  grp.sync();  // sm reusable by the next scan
  return op(wp, exc);
}

// Hillis-Steele rounds one block_exclusive over `nact` threads runs.
__host__ __device__ inline int cta_scan_rounds(int nact) {
  int r = 0;
  while ((1 << r) < nact) ++r;
  return r;
}

// Inclusive scan over the chain's links of a K-field array stored in the
// workspace (ws[(f0 + k) * n + i]), in place. Links not present use identity.
template <int K, bool REVERSE, class Op, class G = CtaGroup>
__device__ void ws_scan(double* ws, int n, int f0, int lpt, Op op, ScanSmem& sm, const G& grp = G{}) {
  const int t = grp.tid();
  const int i0 = t * lpt, i1 = min(n, i0 + lpt);
  Arr<K> agg = op.template identity<K>();
  // local inclusive scan of own links
  for (int s = 0; s < i1 - i0; ++s) {
    const int i = REVERSE ? (i1 - 1 - s) : (i0 + s);
    Arr<K> x;
#pragma unroll
    for (int k = 0; k < K; ++k) x.v[k] = ws[(f0 + k) * n + i];
    agg = op(agg, x);
#pragma unroll
    for (int k = 0; k < K; ++k) ws[(f0 + k) * n + i] = agg.v[k];
  }
  const Arr<K> pre = block_exclusive<K, REVERSE>(agg, op, sm, (n + lpt - 1) / lpt, grp);
  for (int i = i0; i < i1; ++i) {
    Arr<K> x;
#pragma unroll
    for (int k = 0; k < K; ++k) x.v[k] = ws[(f0 + k) * n + i];
    x = op(pre, x);
#pragma unroll
    for (int k = 0; k < K; ++k) ws[(f0 + k) * n + i] = x.v[k];
  }
}

__device__ __forceinline__ void ws_put_sv(double* ws, int n, int f0, int i, const Sv& x) {
  ws[(f0 + 0) * n + i] = x.a.x;
  ws[(f0 + 1) * n + i] = x.a.y;
  ws[(f0 + 2) * n + i] = x.a.z;
  ws[(f0 + 3) * n + i] = x.l.x;
  ws[(f0 + 4) * n + i] = x.l.y;
  ws[(f0 + 5) * n + i] = x.l.z;
}
__device__ __forceinline__ Sv ws_get_sv(const double* ws, int n, int f0, int i) {
  return {mk(ws[(f0 + 0) * n + i], ws[(f0 + 1) * n + i], ws[(f0 + 2) * n + i]),
          mk(ws[(f0 + 3) * n + i], ws[(f0 + 4) * n + i], ws[(f0 + 5) * n + i])};
}
__device__ __forceinline__ void ws_put_se3(double* ws, int n, int f0, int i, const SE3d& T) {
#pragma unroll
  for (int k = 0; k < 9; ++k) ws[(f0 + k) * n + i] = T.R.m[k];
  ws[(f0 + 9) * n + i] = T.p.x;
  ws[(f0 + 10) * n + i] = T.p.y;
  ws[(f0 + 11) * n + i] = T.p.z;
}
__device__ __forceinline__ SE3d ws_get_se3(const double* ws, int n, int f0, int i) {
  SE3d T;
#pragma unroll
  for (int k = 0; k < 9; ++k) T.R.m[k] = ws[(f0 + k) * n + i];
  T.p = mk(ws[(f0 + 9) * n + i], ws[(f0 + 10) * n + i], ws[(f0 + 11) * n + i]);
  return T;
}

// Workspace fields used by the CTA inverse-dynamics stage.
struct IdFields {
  int rel;  // 12: rel_i
  int x;    // 12: X_i
  int v;    // 6:  V_i
  int tmp;  // 6:  scan scratch
  int td;   // 1:  tau_delta_i (out)
};

// Stage: joint transforms rel_i into ws (per link, independent).
template <class G = CtaGroup>
__device__ __forceinline__ void cta_kinematics(const ModelView& mv, const BatchIO& io, int64_t p, int64_t mc,
                                               double* ws, const IdFields& F, int lpt, const G& grp = G{}) {
  const int n = mv.n;
  const int i0 = grp.tid() * lpt, i1 = min(n, i0 + lpt);
  for (int i = i0; i < i1; ++i) {
    const SE3d T = joint_transform(mv.screw(i, mc), mv.screw_iw(i, mc), mv.home_R(i, mc), mv.home_p(i, mc),
                                   io.ld(io.q, i, p));
    ws_put_se3(ws, n, F.rel, i, T);
    ws_put_se3(ws, n, F.x, i, T);
  }
}

// Stage: tau_delta = tau - ID(q, qd, qdd = 0) with gravity as base
// acceleration -g (forward_dynamics.cpp:35-42). Requires rel in ws. Fields
// v and tmp must be adjacent (tmp = v + 6): the (V0, A0) pair scan uses both.
template <class G = CtaGroup>
__device__ inline void cta_bias_torque(const ModelView& mv, const BatchIO& io, int64_t p, int64_t mc, double* ws,
                                const IdFields& F, int lpt, ScanSmem& sm, const G& grp = G{}) {
  const int n = mv.n;
  const int i0 = grp.tid() * lpt, i1 = min(n, i0 + lpt);
  // X_i = rel_i * X_{i-1}
  grp.sync();
  ws_scan<12, false>(ws, n, F.x, lpt, ComposeOp{}, sm, grp);
  grp.sync();
  // base-frame rate twists s_i = Ad(X_i)^{-1} S_i qd_i, then one pair scan
  // gives V0_i and the bias acceleration sum A0_i (PairOp)
  for (int i = i0; i < i1; ++i) {
    const SE3d X = ws_get_se3(ws, n, F.x, i);
    ws_put_sv(ws, n, F.v, i, adinv_apply(X, io.ld(io.qd, i, p) * mv.screw(i, mc)));
    ws_put_sv(ws, n, F.v + 6, i, svzero());
  }
  grp.sync();
  ws_scan<12, false>(ws, n, F.v, lpt, PairOp{}, sm, grp);
  grp.sync();
  const Vec3d g = mv.gravity(mc);
  const Sv Abase = {mk(0, 0, 0), mk(-g.x, -g.y, -g.z)};
  for (int i = i0; i < i1; ++i) {
    const SE3d X = ws_get_se3(ws, n, F.x, i);
    const Sv V = ad_apply(X, ws_get_sv(ws, n, F.v, i));
    const Sv A = ad_apply(X, Abase + ws_get_sv(ws, n, F.v + 6, i));
    const Inertia J = mv.inertia(i, mc);
    const Sv h = inertia_apply(J, V);
    const Sv f = inertia_apply(J, A) + neg_advT_apply(V, h);
    ws_put_sv(ws, n, F.tmp, i, adT_apply(X, f));  // tmp = v + 6: this link's pair was read above
  }
  grp.sync();
  ws_scan<6, true>(ws, n, F.tmp, lpt, AddOp{}, sm, grp);
  grp.sync();
  for (int i = i0; i < i1; ++i) {
    const SE3d X = ws_get_se3(ws, n, F.x, i);
    const Sv Fi = adinvT_apply(X, ws_get_sv(ws, n, F.tmp, i));
    ws[F.td * n + i] = io.ld(io.tau, i, p) - dot(mv.screw(i, mc), Fi);
  }
  grp.sync();
}

}  // namespace pd
