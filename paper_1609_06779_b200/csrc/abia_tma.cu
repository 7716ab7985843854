// ABIA, TMA-pipelined lane-per-chain kernel for batches of independent chains.
//
// Same arithmetic as abia_lane_kernel (abia_common.cuh); what changes is the
// memory path. A CTA owns a tile of 128 consecutive chains (one per thread).
// For every link step of the three passes one elected thread issues TMA tile
// loads (cp.async.bulk.tensor) of that link's model fields for the whole tile
// -- a {128 chains x 1 link x F fields} box of the [field][link][chain] SoA
// model -- plus the tile's q / qdot / tau rows into a 3-stage shared-memory
// ring, completion tracked by mbarrier transaction counts. Threads read their
// chain's values from shared memory while the next two links are in flight,
// so the FP64 pipes are not left waiting on global-memory latency.
//   pass A loads model fields 10..27 (screw, home R, home p) + q, qd
//   pass B loads all 28 model fields + q, qd, tau
//   pass C loads the 13-double records pass B wrote (after a proxy fence)
#include <cuda.h>

#include <cstdlib>

#include "abia_common.cuh"

namespace pd {

namespace {

constexpr int kT = 128;          // chains per CTA
constexpr int kStageFields = 33; // 28 model + q, qd, tau, sin, cos; pass C uses 13
constexpr int kQ = 28, kQD = 29, kTAU = 30, kSIN = 31, kCOS = 32;
constexpr int kSC0 = kRec;       // scratch rows n*kRec + 2*i + {0,1}: (sin, cos) of link i's joint angle

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
  CUtensorMap model_all;  // box {T, 1, 28}
  CUtensorMap model_kin;  // box {T, 1, 18} from field 10
  CUtensorMap q, qd, tau; // box {T, 1}
  CUtensorMap scr;        // box {T, 13}
  CUtensorMap sc;         // box {T, 2}: (sin, cos) rows written by pass A
};

}  // namespace

__device__ __forceinline__ Sv stage_screw(const double* f) {
  return {mk(f[F_SCREW * kT], f[(F_SCREW + 1) * kT], f[(F_SCREW + 2) * kT]),
          mk(f[(F_SCREW + 3) * kT], f[(F_SCREW + 4) * kT], f[(F_SCREW + 5) * kT])};
}
__device__ __forceinline__ SE3d stage_rel(const double* f, double st, double ct) {
  Mat3d HR;
#pragma unroll
  for (int j = 0; j < 9; ++j) HR.m[j] = f[(F_HR + j) * kT];
  return joint_transform_sc(stage_screw(f), HR, mk(f[F_HP * kT], f[(F_HP + 1) * kT], f[(F_HP + 2) * kT]), f[kQ * kT],
                            st, ct);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(bar)) : "memory");
}

// KSTAGES-deep ring; MINB CTAs per SM; HINTS = L2 policy (records evict_last
// + discard after use, last-use streams evict_first).
//
// Synchronisation: full[s] (TMA transaction count) tells consumers a stage
// landed; empty[s] (one arrival per warp) tells the producer (thread 0) that
// every warp is done with it. There is no CTA-wide barrier per link: warps
// drift freely within the ring and only the producer waits for the slowest.
// Pass A stores sin/cos of each joint angle for pass B (one sincos per link);
// the last KSTAGES links of pass A, whose pass-B loads are issued before pass A
// reaches them, keep theirs in registers.
template <int KSTAGES, int MINB, bool HINTS>
__global__ void __launch_bounds__(kT, MINB)
    abia_tma_kernel(const __grid_constant__ Maps maps, ModelView mv, BatchIO io, double* __restrict__ scratch,
                    int64_t scr_ld) {
  static_assert(KSTAGES == 3, "the register hand-off of the last pass-A links assumes 3 stages");
  extern __shared__ __align__(128) double ring[];  // [KSTAGES][kStageFields][kT]
  __shared__ __align__(8) uint64_t full[KSTAGES];
  __shared__ __align__(8) uint64_t empty[KSTAGES];
  const int t = threadIdx.x, lane = t & 31;
  const int n = mv.n;
  const int c0 = blockIdx.x * kT;
  const int64_t p = (int64_t)c0 + t;
  const bool live = p < io.B;
  const int total = 3 * n;
  if (t == 0) {
    for (int s = 0; s < KSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t pol_first = 0, pol_last = 0;
  if (HINTS) {
    pol_first = policy_evict_first();
    pol_last = policy_evict_last();
  }

  // step k: pass A link k (k < n), pass B link 2n-1-k, pass C link k-2n
  auto issue = [&](int k) {
    const int s = k % KSTAGES;
    double* dst = ring + (size_t)s * kStageFields * kT;
    uint64_t* bar = &full[s];
    if (k < n) {  // re-read in pass B: default policy
      mbar_expect_tx(bar, (18 + 2) * kT * 8);
      tma_3d(dst + 10 * kT, &maps.model_kin, c0, k, 10, bar);
      tma_2d(dst + kQ * kT, &maps.q, c0, k, bar);
      tma_2d(dst + kQD * kT, &maps.qd, c0, k, bar);
    } else if (k < 2 * n) {  // last use of the model
      const int i = 2 * n - 1 - k;
      mbar_expect_tx(bar, (28 + 5) * kT * 8);
      if (HINTS) {
        tma_3d_hint(dst, &maps.model_all, c0, i, 0, bar, pol_first);
        tma_2d_hint(dst + kTAU * kT, &maps.tau, c0, i, bar, pol_first);
        tma_2d_hint(dst + kSIN * kT, &maps.sc, c0, 2 * i, bar, pol_first);
      } else {
        tma_3d(dst, &maps.model_all, c0, i, 0, bar);
        tma_2d(dst + kTAU * kT, &maps.tau, c0, i, bar);
        tma_2d(dst + kSIN * kT, &maps.sc, c0, 2 * i, bar);
      }
      tma_2d(dst + kQ * kT, &maps.q, c0, i, bar);
      tma_2d(dst + kQD * kT, &maps.qd, c0, i, bar);
    } else {
      const int i = k - 2 * n;
      mbar_expect_tx(bar, kRec * kT * 8);
      if (HINTS)
        tma_2d_hint(dst, &maps.scr, c0, i * kRec, bar, pol_first);
      else
        tma_2d(dst, &maps.scr, c0, i * kRec, bar);
    }
  };
  // Producer = thread 0: steps [0, KSTAGES) up front; at the end of step k it
  // waits until every warp released step k's stage, then issues step
  // k + KSTAGES into it. Pass-C steps read pass B's records, so they are
  // issued only once every warp released the last pass-B step (2n - 1).
  int next = 0;
  if (t == 0)
    for (; next < min(KSTAGES, min(total, 2 * n)); ++next) issue(next);
  auto after_step = [&](int k) {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[k % KSTAGES]);
    if (t == 0) {
      const int target = k < 2 * n - 1 ? min(2 * n, k + 1 + KSTAGES) : min(total, k + 1 + KSTAGES);
      for (; next < target; ++next) {
        const int prev = next - KSTAGES;  // previous user of the stage
        if (prev >= 0) mbar_wait(&empty[prev % KSTAGES], (uint32_t)((prev / KSTAGES) & 1));
        if (next == 2 * n && prev != 2 * n - 1)
          mbar_wait(&empty[(2 * n - 1) % KSTAGES], (uint32_t)(((2 * n - 1) / KSTAGES) & 1));
        issue(next);
      }
    }
  };

  const int64_t mc = live ? mv.model_of(p) : 0;
  AbiaState st;
  abia_init(st, live ? mv.gravity(mc) : mk(0, 0, 0));
  double s0 = 0, c0r = 1, s1 = 0, c1r = 1, s2 = 0, c2r = 1;  // (sin, cos) of links n-1, n-2, n-3
  int k = 0;
  for (; k < n; ++k) {  // pass A
    const int s = k % KSTAGES;
    mbar_wait(&full[s], (uint32_t)((k / KSTAGES) & 1));
    const double* f = ring + (size_t)s * kStageFields * kT + t;
    const Sv S = stage_screw(f);
    double sn, cs;
    joint_angle_sincos(S, f[kQ * kT], &sn, &cs);
    abia_pass_a(st, stage_rel(f, sn, cs), S, f[kQD * kT]);
    if (k < n - KSTAGES) {
      if (live) {
        double* a = scratch + ((int64_t)n * kSC0 + 2 * k) * scr_ld + p;
        if (HINTS) {
          st_hint(a, sn, pol_last);
          st_hint(a + scr_ld, cs, pol_last);
        } else {
          a[0] = sn;
          a[scr_ld] = cs;
        }
      }
    } else {
      s2 = s1; c2r = c1r; s1 = s0; c1r = c0r; s0 = sn; c0r = cs;
    }
    if (k == n - 1) asm volatile("fence.proxy.async.global;" ::: "memory");  // sin/cos rows -> TMA reads
    after_step(k);
  }
  for (; k < 2 * n; ++k) {  // pass B
    const int s = k % KSTAGES;
    mbar_wait(&full[s], (uint32_t)((k / KSTAGES) & 1));
    const double* f = ring + (size_t)s * kStageFields * kT + t;
    const int i = 2 * n - 1 - k;
    double sn = f[kSIN * kT], cs = f[kCOS * kT];
    if (i == n - 1) { sn = s0; cs = c0r; }
    if (i == n - 2) { sn = s1; cs = c1r; }
    if (i == n - 3) { sn = s2; cs = c2r; }
    Inertia J;
    J.m = f[F_MASS * kT];
    J.c = mk(f[F_COM * kT], f[(F_COM + 1) * kT], f[(F_COM + 2) * kT]);
#pragma unroll
    for (int j = 0; j < 6; ++j) J.I[j] = f[(F_IC + j) * kT];
    double rec[kRec];
    abia_pass_b(st, i, n, stage_rel(f, sn, cs), stage_screw(f), f[kQD * kT], J, f[kTAU * kT], rec);
    if (live) {
#pragma unroll
      for (int j = 0; j < kRec; ++j) {
        double* a = scratch + ((int64_t)i * kRec + j) * scr_ld + p;
        if (HINTS)
          st_hint(a, rec[j], pol_last);
        else
          *a = rec[j];
      }
    }
    if (k == 2 * n - 1) asm volatile("fence.proxy.async.global;" ::: "memory");  // records -> TMA reads
    after_step(k);
  }
  for (; k < total; ++k) {  // pass C
    const int s = k % KSTAGES;
    mbar_wait(&full[s], (uint32_t)((k / KSTAGES) & 1));
    const double* f = ring + (size_t)s * kStageFields * kT + t;
    const int i = k - 2 * n;
    double rec[kRec];
#pragma unroll
    for (int j = 0; j < kRec; ++j) rec[j] = f[j * kT];
    const double qdd = abia_pass_c(st, rec);
    if (live) io.put_qdd(i, p, qdd);
    if (HINTS && t < kRec * (kT * 8 / 128)) {
      // the records of link i are dead: drop their L2 lines without write-back
      const int row = t / (kT * 8 / 128), seg = t % (kT * 8 / 128);
      const double* line = scratch + ((int64_t)i * kRec + row) * scr_ld + c0 + seg * 16;
      if (c0 + seg * 16 + 16 <= io.B) discard_l2(line);
    }
    after_step(k);
  }
  if (live) {
    const int32_t ms = __ldg(mv.mstatus + mc);
    io.status[p] = ms != PD_SLOT_OK ? ms : st.code;
    io.eround[p] = 0;
    io.eindex[p] = ms != PD_SLOT_OK ? __ldg(mv.mrule + mc) : st.eidx;
  }
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

// Kernel variant (tuning experiments): PD_ABIA_VARIANT selects
// 0 = L2 policy hints (default), 2 = no hints.
int abia_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("PD_ABIA_VARIANT");
    v = e ? std::atoi(e) : 0;
  }
  return v;
}

}  // namespace

// Returns false (caller falls back to the plain kernel) when the batch does
// not meet TMA's layout rules: one model per chain, 16-byte aligned bases,
// link strides that are multiples of 16 bytes, 32-bit coordinates.
bool launch_abia_tma(const ModelView& mv, const BatchIO& io, double* scratch, int64_t scr_ld, cudaStream_t s) {
  if (mv.M == 1 || mv.M != io.B) return false;
  if ((io.lds & 1) || (mv.ld & 1) || (scr_ld & 1)) return false;
  if (!aligned16(mv.f) || !aligned16(io.q) || !aligned16(io.qd) || !aligned16(io.tau) || !aligned16(scratch))
    return false;
  if (io.B >= (1ll << 31) || (int64_t)mv.n * kRec >= (1ll << 31)) return false;
  const int n = mv.n;
  Maps maps;
  {
    const cuuint64_t dims[3] = {(cuuint64_t)mv.M, (cuuint64_t)n, (cuuint64_t)F_COUNT};
    const cuuint64_t str[2] = {(cuuint64_t)mv.ld * 8, (cuuint64_t)mv.ld * n * 8};
    const cuuint32_t box_all[3] = {kT, 1, 28}, box_kin[3] = {kT, 1, 18};
    if (!encode(&maps.model_all, mv.f, 3, dims, str, box_all)) return false;
    if (!encode(&maps.model_kin, mv.f, 3, dims, str, box_kin)) return false;
  }
  {
    const cuuint64_t dims[2] = {(cuuint64_t)io.B, (cuuint64_t)n};
    const cuuint64_t str[1] = {(cuuint64_t)io.lds * 8};
    const cuuint32_t box[2] = {kT, 1};
    if (!encode(&maps.q, io.q, 2, dims, str, box)) return false;
    if (!encode(&maps.qd, io.qd, 2, dims, str, box)) return false;
    if (!encode(&maps.tau, io.tau, 2, dims, str, box)) return false;
  }
  {
    const cuuint64_t dims[2] = {(cuuint64_t)io.B, (cuuint64_t)n * kRec};
    const cuuint64_t str[1] = {(cuuint64_t)scr_ld * 8};
    const cuuint32_t box[2] = {kT, kRec};
    if (!encode(&maps.scr, scratch, 2, dims, str, box)) return false;
    const cuuint64_t dims_sc[2] = {(cuuint64_t)io.B, (cuuint64_t)n * 2};
    const cuuint32_t box_sc[2] = {kT, 2};
    if (!encode(&maps.sc, scratch + (size_t)n * kSC0 * scr_ld, 2, dims_sc, str, box_sc)) return false;
  }
  const unsigned blocks = (unsigned)((io.B + kT - 1) / kT);
  auto go = [&](auto kernel, int stages) {
    const size_t smem = (size_t)stages * kStageFields * kT * sizeof(double);
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kernel<<<blocks, kT, smem, s>>>(maps, mv, io, scratch, scr_ld);
  };
  switch (abia_variant()) {
    case 2: go(abia_tma_kernel<3, 2, false>, 3); break;
    default: go(abia_tma_kernel<3, 2, true>, 3); break;  // measured best (profiles/README.md)
  }
  return true;
}

}  // namespace pd
