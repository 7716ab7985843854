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

#include "abia_common.cuh"

namespace pd {

namespace {

constexpr int kT = 128;          // chains per CTA
constexpr int kStages = 3;       // ring depth
constexpr int kStageFields = 32; // 28 model + q, qd, tau (+1 pad); pass C uses 13
constexpr int kQ = 28, kQD = 29, kTAU = 30;

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

struct Maps {
  CUtensorMap model_all;  // box {T, 1, 28}
  CUtensorMap model_kin;  // box {T, 1, 18} from field 10
  CUtensorMap q, qd, tau; // box {T, 1}
  CUtensorMap scr;        // box {T, 13}
};

}  // namespace

__device__ __forceinline__ Sv stage_screw(const double* f) {
  return {mk(f[F_SCREW * kT], f[(F_SCREW + 1) * kT], f[(F_SCREW + 2) * kT]),
          mk(f[(F_SCREW + 3) * kT], f[(F_SCREW + 4) * kT], f[(F_SCREW + 5) * kT])};
}
__device__ __forceinline__ SE3d stage_rel(const double* f) {
  Mat3d HR;
#pragma unroll
  for (int j = 0; j < 9; ++j) HR.m[j] = f[(F_HR + j) * kT];
  return joint_transform(stage_screw(f), HR, mk(f[F_HP * kT], f[(F_HP + 1) * kT], f[(F_HP + 2) * kT]), f[kQ * kT]);
}

__global__ void __launch_bounds__(kT, 2)
    abia_tma_kernel(const __grid_constant__ Maps maps, ModelView mv, BatchIO io, double* __restrict__ scratch,
                    int64_t scr_ld) {
  extern __shared__ __align__(128) double ring[];  // [kStages][kStageFields][kT]
  __shared__ __align__(8) uint64_t full[kStages];
  const int t = threadIdx.x;
  const int n = mv.n;
  const int c0 = blockIdx.x * kT;
  const int64_t p = (int64_t)c0 + t;
  const bool live = p < io.B;
  const int total = 3 * n;
  if (t == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // step k: pass A link k (k < n), pass B link 2n-1-k, pass C link k-2n
  auto issue = [&](int k) {
    const int s = k % kStages;
    double* dst = ring + (size_t)s * kStageFields * kT;
    uint64_t* bar = &full[s];
    if (k < n) {
      mbar_expect_tx(bar, (18 + 2) * kT * 8);
      tma_3d(dst + 10 * kT, &maps.model_kin, c0, k, 10, bar);
      tma_2d(dst + kQ * kT, &maps.q, c0, k, bar);
      tma_2d(dst + kQD * kT, &maps.qd, c0, k, bar);
    } else if (k < 2 * n) {
      const int i = 2 * n - 1 - k;
      mbar_expect_tx(bar, (28 + 3) * kT * 8);
      tma_3d(dst, &maps.model_all, c0, i, 0, bar);
      tma_2d(dst + kQ * kT, &maps.q, c0, i, bar);
      tma_2d(dst + kQD * kT, &maps.qd, c0, i, bar);
      tma_2d(dst + kTAU * kT, &maps.tau, c0, i, bar);
    } else {
      const int i = k - 2 * n;
      mbar_expect_tx(bar, kRec * kT * 8);
      tma_2d(dst, &maps.scr, c0, i * kRec, bar);
    }
  };
  // Producer = thread 0. Steps [0, kStages) are issued up front; at the end
  // of step k (after the CTA barrier freed stage k % kStages) it issues step
  // k + kStages into that stage, so each link's data is requested kStages
  // steps before it is used. Pass-C steps read the records pass B wrote and
  // are only issued once the barrier after the last pass-B step has passed.
  int next = 0;
  auto produce_until = [&](int target) {
    for (; next < target; ++next) issue(next);
  };
  if (t == 0) produce_until(min(kStages, min(total, 2 * n)));

  const int64_t mc = live ? mv.model_of(p) : 0;
  AbiaState st;
  abia_init(st, live ? mv.gravity(mc) : mk(0, 0, 0));
  for (int k = 0; k < total; ++k) {
    const int s = k % kStages;
    mbar_wait(&full[s], (uint32_t)((k / kStages) & 1));
    const double* f = ring + (size_t)s * kStageFields * kT + t;
    if (k < n) {
      abia_pass_a(st, stage_rel(f), stage_screw(f), f[kQD * kT]);
    } else if (k < 2 * n) {
      const int i = 2 * n - 1 - k;
      Inertia J;
      J.m = f[F_MASS * kT];
      J.c = mk(f[F_COM * kT], f[(F_COM + 1) * kT], f[(F_COM + 2) * kT]);
#pragma unroll
      for (int j = 0; j < 6; ++j) J.I[j] = f[(F_IC + j) * kT];
      double rec[kRec];
      abia_pass_b(st, i, n, stage_rel(f), stage_screw(f), f[kQD * kT], J, f[kTAU * kT], rec);
      if (live) {
#pragma unroll
        for (int j = 0; j < kRec; ++j) scratch[((int64_t)i * kRec + j) * scr_ld + p] = rec[j];
      }
      if (k == 2 * n - 1) asm volatile("fence.proxy.async.global;" ::: "memory");  // records -> TMA reads
    } else {
      const int i = k - 2 * n;
      double rec[kRec];
#pragma unroll
      for (int j = 0; j < kRec; ++j) rec[j] = f[j * kT];
      const double qdd = abia_pass_c(st, rec);
      if (live) io.put_qdd(i, p, qdd);
    }
    __syncthreads();  // stage s consumed; at k = 2n-1 also: every record written
    if (t == 0) produce_until(k < 2 * n - 1 ? min(2 * n, k + 1 + kStages) : min(total, k + 1 + kStages));
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
  }
  const size_t smem = (size_t)kStages * kStageFields * kT * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(abia_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const unsigned blocks = (unsigned)((io.B + kT - 1) / kT);
  abia_tma_kernel<<<blocks, kT, smem, s>>>(maps, mv, io, scratch, scr_ld);
  return true;
}

}  // namespace pd
