// ABIA for batches of independent chains, lane per chain, TMA-fed.
//
// Same arithmetic as abia_lane_kernel (abia_common.cuh: three fused passes in
// base coordinates); what differs is the memory path. A CTA owns tiles of KT
// consecutive chains (one per consumer thread). For every link step of the
// three passes TMA tile loads (cp.async.bulk.tensor) bring that link's fields
// for the whole tile -- a {KT chains x 1 link x F fields} box of the
// [field][link][chain] SoA model -- plus the tile's q / qdot / tau rows into
// shared memory, completion tracked by mbarrier transaction counts:
//   pass A: the F_NKIN kinematic fields + q, qd
//   pass B: all F_COUNT model fields + q, qd, tau
//   pass C: the 13-double records pass B wrote (after a proxy fence)
// abia_ring_kernel: a dedicated producer warp streams the steps of all the
// CTA's tiles (persistent CTAs) through one byte ring with per-pass stage
// sizes, so cheap passes run many links ahead and the next tile's pass A
// streams in during this tile's pass C.
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "abia_common.cuh"

namespace pd {

namespace {

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(saddr(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(saddr(bar))
      : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(saddr(bar))
      : "memory");
}

__device__ __forceinline__ void tma_3d_hint(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar,
                                            uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, "
      "%4}], [%5], %6;" ::"r"(saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(saddr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_2d_hint(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                            uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(saddr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_hint(double* addr, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(addr), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void discard_l2(const void* addr) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(addr) : "memory");
}

struct Maps {
  CUtensorMap model_all;  // box {T, 1, F_COUNT}
  CUtensorMap model_kin;  // box {T, 1, F_NKIN} from field F_KIN
  CUtensorMap q, qd, tau; // box {T, 1}
  CUtensorMap scr;        // box {T, 13}
};

}  // namespace

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(bar)) : "memory");
}

// ---------------------------------------------------------------------------
// Ring-buffer variant: same three passes and arithmetic, but the stages are
// sized per pass (pass A 20 rows, pass B 31, pass C 13; a row = one field of
// the KT-chain tile) in one shared-memory byte ring, so the cheap passes run
// many links ahead (up to kSlots steps in flight) instead of a fixed
// 3-stage depth. Pass B recomputes the joint sin/cos instead of reading them
// back (no scratch round trip, no register hand-off of the last links).
// Thread 0 is the producer; it never blocks on a stage it does not need yet:
// before consuming step k it issues up to k (blocking reclaims), after each
// step it issues further ahead only while slots are free (non-blocking).
constexpr int kSlots = 16;
constexpr int kRowsA = F_NKIN + 2, kRowsB = F_COUNT + 3, kRowsC = kRec;

// rows r0.. = the kinematic block F_SW..F_HP: w, vx, vz, 1/w, home quaternion (4), home p (3)
template <int KT>
__device__ __forceinline__ Sv row_screw(const double* f, int r0) {
  return joint_screw(f[r0 * KT], f[(r0 + 1) * KT], f[(r0 + 2) * KT]);
}
template <int KT>
__device__ __forceinline__ SE3d row_rel(const double* f, int r0, const Sv& S, double q, double st, double ct) {
  const Mat3d HR = quat_to_R(f[(r0 + 4) * KT], f[(r0 + 5) * KT], f[(r0 + 6) * KT], f[(r0 + 7) * KT]);
  return joint_transform_sc(S, f[(r0 + 3) * KT], HR, mk(f[(r0 + 8) * KT], f[(r0 + 9) * KT], f[(r0 + 10) * KT]), q,
                            st, ct);
}

// MAXREG caps registers per thread (__maxnreg__) so that the wanted number of
// CTAs fits the SM's 64K registers (e.g. 2 x 160 threads x 200).
// SPLIT: the producer warpgroup gives its registers to the consumers
// (setmaxnreg inside each role's branch, so ptxas allocates each role's code
// with its own budget).
// BIAS: torque-surplus mode -- passes A and B only, pass B reduced to the
// link wrenches, tau_delta written to io.qdd's slot ([link][problem]); no
// records, no pass C, no status.
template <int KT, bool SPLIT = false, bool BIAS = false>
__device__ __forceinline__ void abia_ring_body(const Maps& maps, const ModelView& mv, const BatchIO& io,
                                               double* __restrict__ scratch, int64_t scr_ld, uint32_t cap_rows) {
  static_assert(KT % 16 == 0, "ring rows must stay 128-byte aligned for TMA");
  extern __shared__ __align__(128) double ring[];  // cap_rows x KT doubles
  __shared__ __align__(8) uint64_t full[kSlots];
  __shared__ __align__(8) uint64_t empty[kSlots];
  __shared__ uint32_t vstart[kSlots];  // producer only: virtual ring row of each step in flight
  constexpr int NW = (KT + 31) / 32;   // consumer warps; warp NW is the producer
  const int t = threadIdx.x, lane = t & 31;
  const int n = mv.n;
  const uint32_t total = (BIAS ? 2u : 3u) * (uint32_t)n;
  const int ntiles = (int)((io.B + KT - 1) / KT);
  if (t == 0) {
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();
  auto rows_of = [&](uint32_t k) -> uint32_t { return k < (uint32_t)n ? kRowsA : (k < 2u * n ? kRowsB : kRowsC); };
  // Persistent CTA: tiles blockIdx.x, blockIdx.x + gridDim.x, ... flow through
  // one ring, so the next tile's pass-A loads stream in during this tile's
  // (memory-light) pass C. Steps are numbered gk across the CTA's tiles.
  if (t >= NW * 32) {  // ---- producer warp(s): one elected lane issues every step in order
    if constexpr (SPLIT) asm volatile("setmaxnreg.dec.sync.aligned.u32 24;" ::: "memory");
    if (t == NW * 32) {
      uint32_t vpos = 0, phys = 0, old = 0, gk = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int c0 = tile * KT;
        const uint32_t base = gk;
        for (uint32_t k = 0; k < total; ++k, ++gk) {
          const uint32_t rows = rows_of(k);
          if (phys + rows > cap_rows) {  // wrap: skip the ring's tail
            vpos += cap_rows - phys;
            phys = 0;
          }
          // free the slot, the ring rows, and (pass C) every pass-B step of this tile
          while (gk - old >= (uint32_t)kSlots || (old < gk && vpos + rows - vstart[old % kSlots] > cap_rows) ||
                 (k >= 2u * n && old < base + 2u * n)) {
            mbar_wait(&empty[old % kSlots], (old / kSlots) & 1u);
            ++old;
          }
          double* dst = ring + (size_t)phys * KT;
          uint64_t* bar = &full[gk % kSlots];
          if (k < (uint32_t)n) {  // pass A: kinematic rows 0..F_NKIN-1, q, qd
            mbar_expect_tx(bar, kRowsA * KT * 8);
            if constexpr (SPLIT) {  // 256-chain tiles (the largest batches): the rows would not survive to pass B
              tma_3d_hint(dst, &maps.model_kin, c0, (int)k, F_KIN, bar, pol_first);
              tma_2d_hint(dst + F_NKIN * KT, &maps.q, c0, (int)k, bar, pol_first);
              tma_2d_hint(dst + (F_NKIN + 1) * KT, &maps.qd, c0, (int)k, bar, pol_first);
            } else {
              tma_3d(dst, &maps.model_kin, c0, (int)k, F_KIN, bar);
              tma_2d(dst + F_NKIN * KT, &maps.q, c0, (int)k, bar);
              tma_2d(dst + (F_NKIN + 1) * KT, &maps.qd, c0, (int)k, bar);
            }
          } else if (k < 2u * n) {  // pass B: model rows 0..F_COUNT-1, q, qd, tau (last use)
            const int i = 2 * n - 1 - (int)k;
            mbar_expect_tx(bar, kRowsB * KT * 8);
            tma_3d_hint(dst, &maps.model_all, c0, i, 0, bar, pol_first);
            tma_2d_hint(dst + F_COUNT * KT, &maps.q, c0, i, bar, pol_first);
            tma_2d_hint(dst + (F_COUNT + 1) * KT, &maps.qd, c0, i, bar, pol_first);
            tma_2d_hint(dst + (F_COUNT + 2) * KT, &maps.tau, c0, i, bar, pol_first);
          } else {  // pass C: records of link i
            const int i = (int)k - 2 * n;
            mbar_expect_tx(bar, kRowsC * KT * 8);
            tma_2d_hint(dst, &maps.scr, c0, i * kRec, bar, pol_first);
          }
          vstart[gk % kSlots] = vpos;
          vpos += rows;
          phys += rows;
        }
      }
    }
    return;
  }
  if constexpr (SPLIT) asm volatile("setmaxnreg.inc.sync.aligned.u32 240;" ::: "memory");
  uint32_t cphys = 0, gk = 0;  // consumer's ring position / step counter (mirror the producer's)
  const int tt = t < KT ? t : 0;
  // step k's rows; `ahead` = steps already acquired and not yet released
  auto acquire = [&](uint32_t k, uint32_t ahead = 0) -> const double* {
    const uint32_t rows = rows_of(k);
    if (cphys + rows > cap_rows) cphys = 0;
    const uint32_t off = cphys;
    cphys += rows;
    const uint32_t g = gk + ahead;
    mbar_wait(&full[g % kSlots], (g / kSlots) & 1u);
    return ring + (size_t)off * KT + tt;
  };
  auto release = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[gk % kSlots]);
    ++gk;
  };

  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int c0 = tile * KT;
    const int64_t p = (int64_t)c0 + t;
    const bool live = t < KT && p < io.B;  // lanes past KT (partial last warp) only keep the warp convergent
    const int64_t mc = live ? mv.model_of(p) : 0;
    AbiaState st;
    abia_init(st, live ? mv.gravity(mc) : mk(0, 0, 0));
    uint32_t k = 0;
    for (; k < (uint32_t)n; ++k) {  // pass A
      const double* f = acquire(k);
      const Sv S = row_screw<KT>(f, 0);
      const double q = f[F_NKIN * KT];
      double sn, cs;
      joint_angle_sincos(S, q, &sn, &cs);
      abia_pass_a(st, row_rel<KT>(f, 0, S, q, sn, cs), S, f[(F_NKIN + 1) * KT]);
      release();
    }
    auto link_b = [&](const double* f, uint32_t kk) {
      const int i = 2 * n - 1 - (int)kk;
      const Sv S = row_screw<KT>(f, F_KIN);
      const double q = f[F_COUNT * KT];
      double sn, cs;
      joint_angle_sincos(S, q, &sn, &cs);
      Inertia J;
      J.m = f[F_MASS * KT];
      J.c = mk(f[F_COM * KT], f[(F_COM + 1) * KT], f[(F_COM + 2) * KT]);
#pragma unroll
      for (int j = 0; j < 6; ++j) J.I[j] = f[(F_IC + j) * KT];
      if constexpr (BIAS) {
        const double td = abia_pass_b_bias(st, row_rel<KT>(f, F_KIN, S, q, sn, cs), S, f[(F_COUNT + 1) * KT], J,
                                           f[(F_COUNT + 2) * KT]);
        if (live) io.put_qdd(i, p, td);
        return;
      }
      double rec[kRec];
      abia_pass_b(st, i, n, row_rel<KT>(f, F_KIN, S, q, sn, cs), S, f[(F_COUNT + 1) * KT], J, f[(F_COUNT + 2) * KT],
                  rec, q);
      if (live) {
#pragma unroll
        for (int j = 0; j < kRec; ++j) st_hint(scratch + ((int64_t)i * kRec + j) * scr_ld + p, rec[j], pol_last);
      }
    };
    // pass B two links per wait: both steps' rows are in shared memory before
    // either link computes, so the scheduler can overlap link i-1's
    // independent work (frame, link inertia, wrench) with link i's
    // articulated-inertia chain
    for (; k + 1 < 2u * n; k += 2) {
      const double* fa = acquire(k);
      const double* fb = acquire(k + 1, 1);
      link_b(fa, k);
      link_b(fb, k + 1);
      if (k + 1 == 2u * n - 1) asm volatile("fence.proxy.async.global;" ::: "memory");  // records -> TMA reads
      release();
      release();
    }
    for (; k < 2u * n; ++k) {  // odd n: the last pass-B step
      link_b(acquire(k), k);
      asm volatile("fence.proxy.async.global;" ::: "memory");
      release();
    }
    if constexpr (BIAS) continue;
    for (; k < total; ++k) {  // pass C
      const double* f = acquire(k);
      const int i = (int)k - 2 * n;
      double rec[kRec];
#pragma unroll
      for (int j = 0; j < kRec; ++j) rec[j] = f[j * KT];
      const double qdd = abia_pass_c(st, rec);
      if (live) io.put_qdd(i, p, qdd);
      if (KT % 16 == 0 && t < kRec * (KT / 16)) {  // drop the dead records' L2 lines without write-back
        const int row = t / (KT / 16), seg = t % (KT / 16);
        const double* line = scratch + ((int64_t)i * kRec + row) * scr_ld + c0 + seg * 16;
        if (c0 + seg * 16 + 16 <= io.B) discard_l2(line);
      }
      release();
    }
    if (live) {
      const int32_t ms = __ldg(mv.mstatus + mc);
      io.status[p] = ms != PD_SLOT_OK ? ms : st.code;
      io.eround[p] = 0;
      io.eindex[p] = ms != PD_SLOT_OK ? __ldg(mv.mrule + mc) : st.eidx;
    }
  }
}

template <int KT, int MAXREG>
__global__ void __launch_bounds__((KT + 31) / 32 * 32 + 32) __maxnreg__(MAXREG)
    abia_ring_kernel(const __grid_constant__ Maps maps, ModelView mv, BatchIO io, double* __restrict__ scratch,
                     int64_t scr_ld, uint32_t cap_rows) {
  abia_ring_body<KT>(maps, mv, io, scratch, scr_ld, cap_rows);
}

// The torque surplus tau_delta = tau - ID(q, qd, 0) of every chain through the
// same TMA ring (passes A and B of the ABIA kernel without its articulated
// part), into io.qdd's slot: CFA's pre-pass for large batches.
__global__ void __launch_bounds__(256, 1)
    bias_ring_kernel(const __grid_constant__ Maps maps, ModelView mv, BatchIO io, double* __restrict__ scratch,
                     int64_t scr_ld, uint32_t cap_rows) {
  abia_ring_body<224, false, true>(maps, mv, io, scratch, scr_ld, cap_rows);
}

// 256-chain tiles: eight consumer warps (two warpgroups raised to 240
// registers) and a producer warpgroup lowered to 24 (one working lane), so
// every SMSP carries two consumer warps within the SM's 64K registers
// (384 x 168 at launch = 256 x 240 + 128 x 24).
__global__ void __launch_bounds__(384, 1)
    abia_ring8_kernel(const __grid_constant__ Maps maps, ModelView mv, BatchIO io, double* __restrict__ scratch,
                      int64_t scr_ld, uint32_t cap_rows) {
  abia_ring_body<256, true>(maps, mv, io, scratch, scr_ld, cap_rows);
}

// ---------------------------------------------------------------- host side
namespace {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

bool encode(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides_bytes,
            const cuuint32_t* box) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (cuuint32_t)rank, const_cast<void*>(base), dims, strides_bytes, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

bool encode_maps(Maps& maps, const ModelView& mv, const BatchIO& io, double* scratch, int64_t scr_ld, uint32_t kt,
                 bool records = true) {
  const int n = mv.n;
  {
    const cuuint64_t dims[3] = {(cuuint64_t)mv.M, (cuuint64_t)n, (cuuint64_t)F_COUNT};
    const cuuint64_t str[2] = {(cuuint64_t)mv.ld * 8, (cuuint64_t)mv.ld * n * 8};
    const cuuint32_t box_all[3] = {kt, 1, F_COUNT}, box_kin[3] = {kt, 1, F_NKIN};
    if (!encode(&maps.model_all, mv.f, 3, dims, str, box_all)) return false;
    if (!encode(&maps.model_kin, mv.f, 3, dims, str, box_kin)) return false;
  }
  {
    const cuuint64_t dims[2] = {(cuuint64_t)io.B, (cuuint64_t)n};
    const cuuint64_t str[1] = {(cuuint64_t)io.lds * 8};
    const cuuint32_t box[2] = {kt, 1};
    if (!encode(&maps.q, io.q, 2, dims, str, box)) return false;
    if (!encode(&maps.qd, io.qd, 2, dims, str, box)) return false;
    if (!encode(&maps.tau, io.tau, 2, dims, str, box)) return false;
  }
  if (records) {
    const cuuint64_t dims[2] = {(cuuint64_t)io.B, (cuuint64_t)n * kRec};
    const cuuint64_t str[1] = {(cuuint64_t)scr_ld * 8};
    const cuuint32_t box[2] = {kt, kRec};
    if (!encode(&maps.scr, scratch, 2, dims, str, box)) return false;
  }
  return true;
}

int sm_count() {
  static int c = 0;
  if (!c) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || c <= 0) c = 148;
  }
  return c;
}

// Returns 0 (caller falls back to the plain lane kernel) when the batch does
// not meet TMA's layout rules: one model per chain, 16-byte aligned bases,
// link strides that are multiples of 16 bytes, 32-bit coordinates. Otherwise
// launches the persistent ring kernel and returns its tile size.
//
// Tile size by the makespan estimate over the selection batch `sel_B` (the
// global batch when a caller shards it, so every shard runs the same
// instantiation): with more tiles than SMs the SM throughput is shared by its
// resident CTAs, so a tile costs KT * ctas chain-units per wave; with fewer
// tiles than SMs each tile runs alone and costs KT. The arithmetic per chain
// is the same for every tile size (abia_common.cuh).
//
// `eff` is the measured per-chain throughput of a configuration relative to
// one 224-chain CTA per SM (7 consumer warps): two 96-chain CTAs (2 x 3
// consumer warps, two producer warps) run 10 % slower per chain (c5a, 1M x 64:
// 5.18 ms at 224 x 1, 5.77 ms at 96 x 2; profiles/abia_tile_r2.txt), so they win
// only where they fill SMs a 224-chain tiling would leave idle. One
// 256-chain CTA (abia_ring8_kernel: 8 consumer warps, two per SMSP, with the
// producer warpgroup's registers) moves 6 % more chains per unit time (c5a
// 4.93 -> 4.66 ms; a tile takes 8 % longer for 14 % more chains), which wins
// once the batch spans enough waves for the larger tile to save one.
int abia_ring_tile(int64_t sel_B) {
  struct Cfg { int kt, ctas; double eff; };
  const Cfg cfgs[4] = {{224, 1, 1.0}, {256, 1, 1.06}, {96, 2, 0.9}, {64, 3, 0.85}};
  double best = 1e300;
  int kt = 224;
  for (const Cfg& c : cfgs) {
    const int64_t tiles = (sel_B + c.kt - 1) / c.kt;
    const int64_t slots = (int64_t)sm_count() * c.ctas;
    const double cost = (tiles <= sm_count() ? (double)c.kt : (double)((tiles + slots - 1) / slots) * c.kt * c.ctas) /
                        c.eff;
    if (cost < best) {
      best = cost;
      kt = c.kt;
    }
  }
  return kt;
}

int launch_abia_tma(const ModelView& mv, const BatchIO& io, double* scratch, int64_t scr_ld, int64_t sel_B,
                    unsigned* grid_out, cudaStream_t s) {
  if (mv.M == 1 || mv.M != io.B) return 0;
  if ((io.lds & 1) || (mv.ld & 1) || (scr_ld & 1)) return 0;
  if (!aligned16(mv.f) || !aligned16(io.q) || !aligned16(io.qd) || !aligned16(io.tau) || !aligned16(scratch)) return 0;
  if (io.B >= (1ll << 31) || (int64_t)mv.n * kRec >= (1ll << 31)) return 0;
  const uint32_t kt = (uint32_t)abia_ring_tile(sel_B);
  const int ctas = (kt == 224 || kt == 256) ? 1 : (kt == 96 ? 2 : 3);
  Maps maps;
  if (!encode_maps(maps, mv, io, scratch, scr_ld, kt)) return 0;
  // the ring takes the SM's shared memory
  const size_t smem = (size_t)(220 * 1024 / ctas) / (kt * 8) * (kt * 8);
  const uint32_t cap_rows = (uint32_t)(smem / (kt * 8));
  const int64_t ntiles = (io.B + kt - 1) / kt;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)sm_count() * ctas);  // persistent CTAs
  auto go = [&](auto kernel) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kernel<<<grid, (kt + 31) / 32 * 32 + 32, smem, s>>>(maps, mv, io, scratch, scr_ld, cap_rows);
  };
  if (kt == 256) {
    cudaFuncSetAttribute(abia_ring8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    abia_ring8_kernel<<<grid, 384, smem, s>>>(maps, mv, io, scratch, scr_ld, cap_rows);
  } else if (kt == 224)
    go(abia_ring_kernel<224, 255>);
  else if (kt == 96)
    go(abia_ring_kernel<96, 248>);
  else
    go(abia_ring_kernel<64, 224>);
  if (grid_out) *grid_out = grid;
  return (int)kt;
}

// tau_delta of every chain into io.qdd ([link][problem], stride io.lds) by the
// ring kernel's passes A and B (bias_ring_kernel); false when the batch does
// not meet TMA's layout rules (the caller then runs the lane pre-pass).
bool launch_bias_tma(const ModelView& mv, const BatchIO& io, cudaStream_t s) {
  if (mv.M == 1 || mv.M != io.B) return false;
  if ((io.lds & 1) || (mv.ld & 1)) return false;
  if (!aligned16(mv.f) || !aligned16(io.q) || !aligned16(io.qd) || !aligned16(io.tau)) return false;
  if (io.B >= (1ll << 31)) return false;
  constexpr uint32_t kt = 224;
  Maps maps;
  if (!encode_maps(maps, mv, io, nullptr, 0, kt, false)) return false;
  const size_t smem = (size_t)(220 * 1024) / (kt * 8) * (kt * 8);
  const uint32_t cap_rows = (uint32_t)(smem / (kt * 8));
  const int64_t ntiles = (io.B + kt - 1) / kt;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)sm_count());
  cudaFuncSetAttribute(bias_ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  bias_ring_kernel<<<grid, 256, smem, s>>>(maps, mv, io, nullptr, 0, cap_rows);
  return true;
}

}  // namespace pd
