// C-ABI of libpardyn_b200.so (include/pardyn_c.h): context, model upload and
// packing, layout transposes for host buffers, kernel dispatch, reference
// error messages. No CPU fallback: every solve runs on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "frames.cuh"

namespace pd {
void launch_abia(const ModelView& mv, const BatchIO& io, double* scratch, cudaStream_t s);
int launch_abia_tma(const ModelView& mv, const BatchIO& io, double* scratch, int64_t scr_ld, int64_t sel_B,
                    unsigned* grid_out, cudaStream_t s);
void launch_abia_cta(const ModelView& mv, const BatchIO& io, double* gws, int64_t gws_slots, cudaStream_t s);
size_t abia_cta_workspace_bytes(int n);
int abia_scratch_doubles_per_link();
void launch_invdyn(const ModelView& mv, const BatchIO& io, cudaStream_t s);
void launch_cfa(const ModelView& mv, const BatchIO& io, double* gws, int64_t gws_slots, cudaStream_t s,
                const double* td_pre);
void launch_tau_surplus(const ModelView& mv, const BatchIO& io, double* td, cudaStream_t s);
bool launch_bias_tma(const ModelView& mv, const BatchIO& io, cudaStream_t s);
void launch_cfa_ws(const ModelView& mv, const BatchIO& io, int sm_count, cudaStream_t s);
bool cfa_ws_fits(int n);
void launch_bidiag6(const double* coupling, const double* rhs, double* x, int64_t batch, int n, int upper,
                    cudaStream_t s);
bool launch_bidiag(int dim, const double* coupling, const double* rhs, double* x, int64_t batch, int n, int upper,
                   cudaStream_t s);
bool launch_oee_block(int b, int m, const double* diag, const double* upper, const double* rhs, double* x,
                      int64_t batch, int n, int32_t* status, int32_t* eround, int32_t* eindex, cudaStream_t s);
bool launch_oee_rounds(int b, int m, const double* diag, const double* coupling, const double* rhs, int64_t batch,
                       int n, int distance, int round0, int nrounds, double* diag_out, double* coupling_out,
                       double* rhs_out, int32_t* status, int32_t* eround, int32_t* eindex, cudaStream_t s);
bool cfa_coop_path(int n, int64_t batch);
void launch_cfa_coop(const ModelView& mv, const BatchIO& io, double* gws, int* bad, int sm_count, cudaStream_t s);
size_t cfa_workspace_bytes(int n);
void launch_jsiia(const ModelView& mv, const BatchIO& io, double* gws, int64_t gws_slots, int sm_count,
                  int64_t sel_B, cudaStream_t s);
bool jsiia_smem_path(int n);
bool launch_jsiia_dmma(const ModelView& mv, const double* mcl, const BatchIO& io, cudaStream_t s);
int jsiia_warps(int n, int64_t batch, int sm_count);
size_t jsiia_workspace_bytes(int n);
struct IdOpts {
  double bv[6], ba[6], tip[6];
  int gravity;
};
void launch_idyn(const ModelView& mv, const BatchIO& io, const IdOpts& o, const double* raw, double* vel, double* acc,
                 double* frc, cudaStream_t s);
bool jsiia_coop_path(int n, int64_t batch);
void launch_workload_chains(uint64_t cell, int n, int64_t g0, int64_t count, double* d_links, cudaStream_t s);
void launch_validate_models(const double* raw, int n, int64_t M, int32_t* status, int32_t* rule, cudaStream_t s);
void launch_jsiia_coop(const ModelView& mv, const BatchIO& io, double* gws, int sm_count, int64_t sel_B,
                       cudaStream_t s);
void launch_jsi(const ModelView& mv, const BatchIO& io, double* gws, int64_t gws_slots, int sm_count, double* d_M,
                cudaStream_t s);
}  // namespace pd

using namespace pd;

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct pd_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int sm_count = 148;
  // models
  int32_t n_links = 0;
  int64_t n_models = 0;
  int64_t model_ld = 0;
  DevBuf model, gravity, mstatus, mrule, raw;
  std::vector<int32_t> h_mstatus, h_mrule;  // host copy of the upload validation
  // the last host model set (kept when <= 64 MiB): an identical pd_set_models
  // -- the drop-in's single-chain calls re-send the same chain every call --
  // skips the upload, validation and packing
  std::vector<double> last_links, last_grav;
  bool models_cached = false;
  DevBuf model_cl;        // link-fastest copy [chain][field][link] for warp-per-chain kernels
  bool model_cl_valid = false;
  // scratch
  DevBuf states;  // link-state outputs and their host-order staging
  DevBuf cfa_td;  // tau_delta [link][problem] for the batched CFA path
  DevBuf abia_scratch, cta_ws, slots, io_q, io_qd, io_tau, io_qdd, io_status;
  // host-buffer path: copy-in / copy-out streams and per-chunk events
  static constexpr int kMaxChunks = 16;
  int32_t* host_status = nullptr;  // pinned staging for slot status
  int32_t* h_flag = nullptr;       // pinned: OR of the slot codes of the last host-buffer call
  DevBuf d_flag;
  size_t host_status_n = 0;
  cudaStream_t cp_in = nullptr, cp_out = nullptr;
  cudaEvent_t ev_entry = nullptr, ev_in[kMaxChunks] = {}, ev_out[kMaxChunks] = {};
  int64_t launches = 0;
  std::string last_error;
  // variant selection: batch size the kernel choice is made for (0 = each
  // call's own batch; a sharding caller sets the global batch so every shard
  // runs the same instantiations and the results are partition independent)
  int64_t selection_batch = 0;
  // what the last forward-dynamics call ran (pd_last_variant / pd_last_trace)
  std::string last_variant;
  pd_exec_trace last_trace{};
};

namespace {

pd_status cuda_fail(pd_ctx* c, cudaError_t e, const char* where) {
  c->last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return PD_CUDA_ERROR;
}

#define PD_CUDA(call)                                         \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call);  \
  } while (0)

// raw [M][n][31] -> packed SoA [F_COUNT][n][M] in joint-aligned frames;
// gravity [M][3] -> [3][M]
__global__ void pack_models_kernel(const double* __restrict__ raw, const double* __restrict__ graw, int n,
                                   int64_t M, int64_t ld, double* __restrict__ out, double* __restrict__ gout) {
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (m >= M) return;
  const double* r = raw + ((int64_t)m * n + i) * PD_LINK_FIELDS;
  auto put = [&](int f, double v) { out[((int64_t)f * n + i) * ld + m] = v; };
  double Q[9], Qp[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, sz[3], dummy[3];
  joint_frame(r + 13, Q, sz);
  if (i > 0) joint_frame(r - PD_LINK_FIELDS + 13, Qp, dummy);
  put(F_MASS, r[0]);
  // com' = Q c
  for (int k = 0; k < 3; ++k) put(F_COM + k, Q[3 * k] * r[1] + Q[3 * k + 1] * r[2] + Q[3 * k + 2] * r[3]);
  // Ic' = Q Ic Q^T from the lower triangle of Ic (what LLT / the assembled blocks read)
  double I[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) I[3 * a + b] = a >= b ? r[4 + 3 * a + b] : r[4 + 3 * b + a];
  double T[9];  // Q Ic
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) T[3 * a + b] = Q[3 * a] * I[b] + Q[3 * a + 1] * I[3 + b] + Q[3 * a + 2] * I[6 + b];
  const int sidx[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
  for (int k = 0; k < 6; ++k) {
    const int a = sidx[k][0], b = sidx[k][1];
    put(F_IC + k, T[3 * a] * Q[3 * b] + T[3 * a + 1] * Q[3 * b + 1] + T[3 * a + 2] * Q[3 * b + 2]);
  }
  // S' = (0, 0, |w|, v'x, 0, v'z): the free components and 1/|w|
  put(F_SW, sz[0]);
  put(F_SVX, sz[1]);
  put(F_SVZ, sz[2]);
  put(F_SIW, sz[0] * sz[0] < 1e-24 ? 0.0 : 1.0 / sz[0]);
  // home' = (Q R_h Qp^T, Q p_h), the rotation stored as a unit quaternion
  const double* Rh = r + 19;
  double U[9];  // Q R_h
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) U[3 * a + b] = Q[3 * a] * Rh[b] + Q[3 * a + 1] * Rh[3 + b] + Q[3 * a + 2] * Rh[6 + b];
  double H[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) H[3 * a + b] = U[3 * a] * Qp[3 * b] + U[3 * a + 1] * Qp[3 * b + 1] + U[3 * a + 2] * Qp[3 * b + 2];
  // as a unit quaternion (Shepperd: the largest of 4w^2, 4x^2, 4y^2, 4z^2 is the pivot)
  double qw, qx, qy, qz;
  const double tr = H[0] + H[4] + H[8];
  if (tr >= H[0] && tr >= H[4] && tr >= H[8]) {
    const double s = 2.0 * sqrt(fmax(1.0 + tr, 0.0));
    qw = 0.25 * s; qx = (H[7] - H[5]) / s; qy = (H[2] - H[6]) / s; qz = (H[3] - H[1]) / s;
  } else if (H[0] >= H[4] && H[0] >= H[8]) {
    const double s = 2.0 * sqrt(fmax(1.0 + H[0] - H[4] - H[8], 0.0));
    qw = (H[7] - H[5]) / s; qx = 0.25 * s; qy = (H[1] + H[3]) / s; qz = (H[2] + H[6]) / s;
  } else if (H[4] >= H[8]) {
    const double s = 2.0 * sqrt(fmax(1.0 + H[4] - H[0] - H[8], 0.0));
    qw = (H[2] - H[6]) / s; qx = (H[1] + H[3]) / s; qy = 0.25 * s; qz = (H[5] + H[7]) / s;
  } else {
    const double s = 2.0 * sqrt(fmax(1.0 + H[8] - H[0] - H[4], 0.0));
    qw = (H[3] - H[1]) / s; qx = (H[2] + H[6]) / s; qy = (H[5] + H[7]) / s; qz = 0.25 * s;
  }
  const double qn = 1.0 / sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
  put(F_HQ, qw * qn);
  put(F_HQ + 1, qx * qn);
  put(F_HQ + 2, qy * qn);
  put(F_HQ + 3, qz * qn);
  for (int k = 0; k < 3; ++k) put(F_HP + k, Q[3 * k] * r[28] + Q[3 * k + 1] * r[29] + Q[3 * k + 2] * r[30]);
  if (i == 0)
    for (int k = 0; k < 3; ++k) gout[(int64_t)k * M + m] = graw[m * 3 + k];
}

// OR of the slot codes into *flag (non-zero iff some slot failed).
__global__ void any_status_kernel(const int32_t* __restrict__ st, int64_t n, int32_t* __restrict__ flag) {
  int32_t acc = 0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    acc |= st[k];
  acc = __reduce_or_sync(0xffffffffu, acc);
  if ((threadIdx.x & 31) == 0 && acc) atomicOr(flag, acc);
}

// [field][link][chain] (stride ld) -> [chain][field][link]
__global__ void repack_link_fastest_kernel(const double* __restrict__ in, int n, int64_t M, int64_t ld,
                                           double* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)M * F_COUNT * n;
  if (idx >= total) return;
  const int i = (int)(idx % n);
  const int f = (int)((idx / n) % F_COUNT);
  const int64_t m = idx / ((int64_t)n * F_COUNT);
  out[idx] = in[((int64_t)f * n + i) * ld + m];
}

// [rows][cols] (row stride ld_in) -> [cols][rows] (row stride ld_out)
// Tiles enumerated on grid.x (column tile fastest): a batch-sized dimension
// on grid.y would cap at 65535 tiles.
__global__ void transpose_kernel(const double* __restrict__ in, double* __restrict__ out, int64_t rows, int64_t cols,
                                 int64_t ld_in, int64_t ld_out) {
  __shared__ double tile[32][33];
  const int64_t ctiles = (cols + 31) / 32;
  const int64_t c0 = ((int64_t)blockIdx.x % ctiles) * 32, r0 = ((int64_t)blockIdx.x / ctiles) * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[k][threadIdx.x] = in[r * ld_in + c];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c = c0 + k, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * ld_out + r] = tile[threadIdx.x][k];
  }
}

// Three same-shaped transposes (q, qdot, tau of a chunk) in one launch.
__global__ void transpose3_kernel(const double* __restrict__ a0, const double* __restrict__ a1,
                                  const double* __restrict__ a2, double* __restrict__ b0, double* __restrict__ b1,
                                  double* __restrict__ b2, int64_t rows, int64_t cols, int64_t ld_in, int64_t ld_out) {
  __shared__ double tile[32][33];
  const double* in = blockIdx.y == 0 ? a0 : (blockIdx.y == 1 ? a1 : a2);
  double* out = blockIdx.y == 0 ? b0 : (blockIdx.y == 1 ? b1 : b2);
  const int64_t ctiles = (cols + 31) / 32;
  const int64_t c0 = ((int64_t)blockIdx.x % ctiles) * 32, r0 = ((int64_t)blockIdx.x / ctiles) * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[k][threadIdx.x] = in[r * ld_in + c];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c = c0 + k, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * ld_out + r] = tile[threadIdx.x][k];
  }
}

void launch_transpose3(pd_ctx* ctx, const double* a0, const double* a1, const double* a2, double* b0, double* b1,
                       double* b2, int64_t rows, int64_t cols, int64_t ld_in, int64_t ld_out) {
  dim3 grid((unsigned)(((cols + 31) / 32) * ((rows + 31) / 32)), 3);
  transpose3_kernel<<<grid, dim3(32, 8), 0, ctx->stream>>>(a0, a1, a2, b0, b1, b2, rows, cols, ld_in, ld_out);
  ctx->launches++;
}

void launch_transpose(pd_ctx* ctx, const double* in, double* out, int64_t rows, int64_t cols, int64_t ld_in,
                      int64_t ld_out) {
  dim3 grid((unsigned)(((cols + 31) / 32) * ((rows + 31) / 32)));
  transpose_kernel<<<grid, dim3(32, 8), 0, ctx->stream>>>(in, out, rows, cols, ld_in, ld_out);
  ctx->launches++;
}

// View of models [m0, m0 + count) (count = batch of a sub-range; a shared
// model is never offset).
ModelView model_view(const pd_ctx* c, int64_t m0 = 0, int64_t count = -1) {
  ModelView mv;
  const bool shared = c->n_models == 1;
  if (shared) m0 = 0;
  mv.f = c->model.as<double>() + m0;
  mv.g = c->gravity.as<double>() + m0;
  mv.mstatus = c->mstatus.as<int32_t>() + m0;
  mv.mrule = c->mrule.as<int32_t>() + m0;
  mv.fcl = nullptr;
  mv.n = c->n_links;
  mv.M = shared ? 1 : (count >= 0 ? count : c->n_models - m0);
  mv.ld = c->model_ld;
  mv.gld = c->n_models;
  return mv;
}

int64_t cta_slots(pd_ctx* ctx, size_t ws_bytes, int64_t batch) {
  const size_t budget = (size_t)2 << 30;  // 2 GiB of global workspace at most
  int64_t slots = (int64_t)std::max<size_t>(1, budget / std::max<size_t>(ws_bytes, 1));
  return std::min<int64_t>(slots, batch);
}

// Builds the link-fastest model copy once per model set (CTA/warp-per-chain kernels).
cudaError_t ensure_model_cl(pd_ctx* ctx) {
  if (ctx->model_cl_valid) return cudaSuccess;
  const int n = ctx->n_links;
  const int64_t total = ctx->n_models * F_COUNT * (int64_t)n;
  cudaError_t e = ctx->model_cl.ensure(sizeof(double) * total);
  if (e != cudaSuccess) return e;
  repack_link_fastest_kernel<<<(unsigned)((total + 255) / 256), 256, 0, ctx->stream>>>(
      ctx->model.as<double>(), n, ctx->n_models, ctx->model_ld, ctx->model_cl.as<double>());
  ctx->launches++;
  ctx->model_cl_valid = true;
  return cudaGetLastError();
}

int ceil_log2_host(int64_t n) {
  int r = 0;
  while ((int64_t(1) << r) < n) ++r;
  return r;
}

// Structure of a CTA-per-chain variant's link-level stages: T threads hold
// ceil(n / lpt) groups of lpt consecutive links; every CTA scan runs
// ceil_log2(groups) Hillis-Steele rounds (cta_common.cuh block_exclusive) after
// a local walk of lpt links.
struct CtaShape {
  int lpt, groups;
};
CtaShape cta_shape(int n, int nt) {
  const int lpt = (n + nt - 1) / nt;
  return {lpt, (n + lpt - 1) / lpt};
}
int cta_threads(int n) { return std::min(256, (n + 31) / 32 * 32); }

void note_variant(pd_ctx* ctx, std::string name, int stages, int seq, int rounds, int oee) {
  ctx->last_variant = std::move(name);
  ctx->last_trace.parallel_link_stages = stages;
  ctx->last_trace.longest_sequential_link_chain = seq;
  ctx->last_trace.scan_rounds_max = rounds;
  ctx->last_trace.oee_rounds = oee;
}

enum Route { ROUTE_AUTO = 0, ROUTE_LOG_DEPTH = 1 };

// Problems [m0, m0 + batch) of the model set (m0 > 0: one chunk of a larger
// host-buffer call; the caller checked the full batch against the models).
// Kernel choice depends on (algo, n, selection batch, route) only:
//   ROUTE_AUTO       the fastest variant for the batch;
//   ROUTE_LOG_DEPTH  the CTA-per-chain variants whose recursions run as
//                    log-depth scans / OEE rounds -- what a traced
//                    single-problem call runs, so ExecTrace
//                    describes the parallel structure the reference's
//                    counters describe (trace.hpp:24-39).
pd_status run_device(pd_ctx* ctx, pd_algo algo, int64_t batch, int64_t lds, const double* q, const double* qd,
                     const double* tau, double* qdd, int32_t* st, int32_t* er, int32_t* ei, int64_t m0 = 0,
                     int64_t sel_batch = 0, Route route = ROUTE_AUTO) {
  if (ctx->n_models <= 0 || ctx->n_links <= 0) {
    ctx->last_error = "forward dynamics: no models set (pd_set_models)";
    return PD_INVALID_ARGUMENT;
  }
  if (ctx->n_models != 1 && m0 + batch > ctx->n_models) {
    ctx->last_error = "forward dynamics: batch must equal the number of models (or use one shared model)";
    return PD_INVALID_ARGUMENT;
  }
  if (batch == 0) return PD_OK;
  const int n = ctx->n_links;
  const int64_t selB = sel_batch > 0 ? sel_batch : (ctx->selection_batch > 0 ? ctx->selection_batch : batch);
  if (!st || !er || !ei) {  // internal scratch only for the slot arrays the caller did not pass
    PD_CUDA(ctx->io_status.ensure(sizeof(int32_t) * 3 * batch));
    int32_t* scr = ctx->io_status.as<int32_t>();
    st = st ? st : scr;
    er = er ? er : scr + batch;
    ei = ei ? ei : scr + 2 * batch;
  }
  BatchIO io{q, qd, tau, qdd, st, er, ei, batch, lds};
  ModelView mv = model_view(ctx, m0, batch);
  const size_t cl_off = ctx->n_models == 1 ? 0 : (size_t)m0 * F_COUNT * n;  // link-fastest copy offset
  const int L = ceil_log2_host(n);
  switch (algo) {
    case PD_ABIA: {
      // long chains in small batches (or a traced call): CTA per chain --
      // parallel kinematics and bias torque, sequential articulated
      // recursion; otherwise lane per chain
      if (route == ROUTE_LOG_DEPTH || (n >= 64 && selB <= 2 * ctx->sm_count)) {
        PD_CUDA(ensure_model_cl(ctx));
        mv.fcl = ctx->model_cl.as<double>() + cl_off;
        const size_t wsb = abia_cta_workspace_bytes(n);
        int64_t slots = 0;
        if (wsb > 200 * 1024) {
          slots = cta_slots(ctx, wsb, batch);
          PD_CUDA(ctx->cta_ws.ensure(wsb * slots));
        }
        launch_abia_cta(mv, io, ctx->cta_ws.as<double>(), slots, ctx->stream);
        ctx->launches += slots ? (batch + slots - 1) / slots : 1;
        const CtaShape cs = cta_shape(n, cta_threads(n));
        // stages: kinematics, 5 bias-torque maps, S0 / J0; one thread walks the
        // articulated recursion over all n links (forward_dynamics.cpp:120-163)
        note_variant(ctx, std::string("abia_cta_kernel<") + (slots ? "global" : "smem") + ">", 7, n,
                     ceil_log2_host(cs.groups), 0);
        break;
      }
      const int64_t scr_ld = (batch + 31) / 32 * 32;
      PD_CUDA(ctx->abia_scratch.ensure(sizeof(double) * abia_scratch_doubles_per_link() * (size_t)n * scr_ld));
      unsigned grid = 0;
      const int kt = launch_abia_tma(mv, io, ctx->abia_scratch.as<double>(), scr_ld, selB, &grid, ctx->stream);
      if (kt)
        note_variant(ctx, "abia_ring_kernel<" + std::to_string(kt) + "> grid " + std::to_string(grid) + " tiles " +
                              std::to_string((batch + kt - 1) / kt), 0, n, 0, 0);
      else {
        launch_abia(mv, io, ctx->abia_scratch.as<double>(), ctx->stream);
        note_variant(ctx, "abia_lane_kernel", 0, n, 0, 0);
      }
      ctx->launches++;
      break;
    }
    case PD_CFA: {
      PD_CUDA(ensure_model_cl(ctx));
      mv.fcl = ctx->model_cl.as<double>() + cl_off;
      const size_t wsb = cfa_workspace_bytes(n);
      const CtaShape cs = cta_shape(n, cta_threads(n));
      if (cfa_coop_path(n, selB)) {  // long chain(s): CTA prologue + grid-wide OEE
        PD_CUDA(ctx->cta_ws.ensure(wsb * batch + 64));
        int* bad = reinterpret_cast<int*>(ctx->cta_ws.as<char>() + wsb * batch);
        launch_cfa_coop(mv, io, ctx->cta_ws.as<double>(), bad, ctx->sm_count, ctx->stream);
        ctx->launches += 2;
        note_variant(ctx, "cfa_cta_kernel<global, prologue> + cfa_oee_coop", 9, cs.lpt > 1 ? cs.lpt : 0,
                     ceil_log2_host(cs.groups), L);
        break;
      }
      int64_t slots = 0;
      if (n > 256 && wsb > 220 * 1024) {
        slots = cta_slots(ctx, wsb, batch);
        PD_CUDA(ctx->cta_ws.ensure(wsb * slots));
        ctx->launches += (batch + slots - 1) / slots;
      } else {
        ctx->launches++;
      }
      if (route == ROUTE_AUTO && cfa_ws_fits(n) && selB >= 2 * (int64_t)ctx->sm_count &&
          selB < 128 * (int64_t)ctx->sm_count) {
        // long chains, enough of them to keep every SM on two: the
        // warp-specialised kernel overlaps chain k+1's prologue with chain k's OEE
        launch_cfa_ws(mv, io, ctx->sm_count, ctx->stream);
        ctx->launches++;
        note_variant(ctx, "cfa_ws_kernel", 9, cs.lpt > 1 ? cs.lpt : 0, ceil_log2_host(cs.groups), L);
        break;
      }
      // large batches: tau_delta by a lane-per-chain pass first (sequential
      // recurrences, no CTA-wide scans); small batches keep the CTA scans
      const double* td_pre = nullptr;
      bool td_ring = false;
      if (route == ROUTE_AUTO && selB >= 128 * (int64_t)ctx->sm_count) {  // >= 4 warps of chains per SM
        PD_CUDA(ctx->cfa_td.ensure(sizeof(double) * (size_t)n * io.lds));
        // the ABIA ring kernel's passes A and B (TMA-streamed, base frame)
        // when the layout allows, else the lane pre-pass
        BatchIO tio = io;
        tio.qdd = ctx->cfa_td.as<double>();
        td_ring = launch_bias_tma(model_view(ctx, m0, batch), tio, ctx->stream);
        if (!td_ring) launch_tau_surplus(model_view(ctx, m0, batch), io, ctx->cfa_td.as<double>(), ctx->stream);
        ctx->launches++;
        td_pre = ctx->cfa_td.as<double>();
      }
      const char* kname = n <= 256 ? "cfa_row_kernel" : (slots ? "cfa_cta_kernel<global>" : "cfa_cta_kernel<smem>");
      launch_cfa(mv, io, ctx->cta_ws.as<double>(), slots, ctx->stream, td_pre);
      if (td_pre)  // tau_delta walked sequentially per chain; operators, OEE and extraction per row
        note_variant(ctx, std::string(td_ring ? "bias_ring_kernel + " : "tau_surplus_lane_kernel + ") + kname, 3, n,
                     0, L);
      else
        note_variant(ctx, kname, 9, cs.lpt > 1 ? cs.lpt : 0, ceil_log2_host(cs.groups), L);
      break;
    }
    case PD_JSIIA: {
      PD_CUDA(ensure_model_cl(ctx));
      mv.fcl = ctx->model_cl.as<double>() + cl_off;
      if (n <= 64 && route == ROUTE_AUTO) {  // warp per chain, M and its Cholesky on the FP64 tensor cores
        launch_jsiia_dmma(mv, mv.fcl, io, ctx->stream);
        ctx->launches++;
        const int lpl = (n + 31) / 32;  // links per lane; warp-shuffle scans of 5 rounds
        note_variant(ctx, "jsiia_dmma_kernel", 5, lpl > 1 ? lpl : 0, 5, 0);
        break;
      }
      const size_t wsb = jsiia_workspace_bytes(n);
      const int nt = 32 * jsiia_warps(n, selB, ctx->sm_count);
      const CtaShape cs = cta_shape(n, nt);
      if (jsiia_coop_path(n, selB)) {  // long chain(s): grid-wide Cholesky
        PD_CUDA(ctx->cta_ws.ensure(wsb * batch));
        launch_jsiia_coop(mv, io, ctx->cta_ws.as<double>(), ctx->sm_count, selB, ctx->stream);
        ctx->launches += 3;
        note_variant(ctx, "jsiia_tiled_kernel<global, prologue> + jsiia_factor_coop + jsiia_solve_wide", 6,
                     cs.lpt > 1 ? cs.lpt : 0, ceil_log2_host(cs.groups), 0);
        break;
      }
      int64_t slots = 0;
      if (!jsiia_smem_path(n)) {
        slots = cta_slots(ctx, wsb, batch);
        PD_CUDA(ctx->cta_ws.ensure(wsb * slots));
        ctx->launches += (batch + slots - 1) / slots;
      } else {
        ctx->launches++;
      }
      launch_jsiia(mv, io, ctx->cta_ws.as<double>(), slots, ctx->sm_count, selB, ctx->stream);
      note_variant(ctx, std::string("jsiia_tiled_kernel<") + (slots ? "global" : "smem") + ">", 6,
                   cs.lpt > 1 ? cs.lpt : 0, ceil_log2_host(cs.groups), 0);
      break;
    }
    default:
      ctx->last_error = "forward_dynamics: unknown algorithm";
      return PD_INVALID_ARGUMENT;
  }
  PD_CUDA(cudaGetLastError());
  return PD_OK;
}

// 8 independent DFMA chains per thread; nothing but FP64 FMAs in the loop.
__global__ void fp64_probe_kernel(double* out, int iters, double seed) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = seed + threadIdx.x * 1e-7 + k;
  const double b = 0.999999999, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;  // keep the chain alive
}

}  // namespace

extern "C" {

pd_status pd_probe_fp64_peak(pd_ctx* ctx, double* tflops, double* elapsed_ms) {
  if (!ctx) return PD_INVALID_ARGUMENT;
  PD_CUDA(cudaSetDevice(ctx->device));
  PD_CUDA(ctx->slots.ensure(64));
  const int threads = 256, blocks = ctx->sm_count * 8, iters = 4096;
  cudaEvent_t e0, e1;
  PD_CUDA(cudaEventCreate(&e0));
  PD_CUDA(cudaEventCreate(&e1));
  fp64_probe_kernel<<<blocks, threads, 0, ctx->stream>>>(ctx->slots.as<double>(), iters, 1.0);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    PD_CUDA(cudaEventRecord(e0, ctx->stream));
    fp64_probe_kernel<<<blocks, threads, 0, ctx->stream>>>(ctx->slots.as<double>(), iters, 1.0 + r);
    PD_CUDA(cudaEventRecord(e1, ctx->stream));
    PD_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    PD_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    best = std::min(best, ms);
  }
  ctx->launches += 6;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double flops = 2.0 * 8.0 * iters * (double)threads * blocks;
  if (tflops) *tflops = flops / (best * 1e-3) / 1e12;
  if (elapsed_ms) *elapsed_ms = best;
  return PD_OK;
}

int pd_abi_version(void) { return PD_ABI_VERSION; }

const char* pd_status_string(pd_status s) {
  switch (s) {
    case PD_OK: return "ok";
    case PD_INVALID_ARGUMENT: return "invalid argument";
    case PD_MODEL_ERROR: return "model error";
    case PD_DYNAMICS_ERROR: return "dynamics error";
    case PD_SINGULAR_BLOCK: return "singular block";
    case PD_CUDA_ERROR: return "CUDA error";
    case PD_NO_DEVICE: return "no CUDA device";
    case PD_INTERNAL: return "internal error";
  }
  return "unknown status";
}

pd_status pd_create(pd_ctx** out, int device) {
  if (!out) return PD_INVALID_ARGUMENT;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return PD_NO_DEVICE;
  if (device < 0 || device >= count) return PD_NO_DEVICE;
  pd_ctx* ctx = new pd_ctx();
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete ctx;
    return PD_CUDA_ERROR;
  }
  cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
  ctx->stream = ctx->own_stream;
  *out = ctx;
  return PD_OK;
}

void pd_destroy(pd_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (DevBuf* b : {&ctx->model, &ctx->gravity, &ctx->mstatus, &ctx->mrule, &ctx->raw, &ctx->abia_scratch, &ctx->cta_ws,
                    &ctx->slots, &ctx->io_q, &ctx->io_qd, &ctx->io_tau, &ctx->io_qdd, &ctx->io_status, &ctx->model_cl,
                    &ctx->states, &ctx->cfa_td, &ctx->d_flag})
    b->release();
  if (ctx->cp_in) {
    cudaStreamSynchronize(ctx->cp_in);
    cudaStreamSynchronize(ctx->cp_out);
    cudaStreamDestroy(ctx->cp_in);
    cudaStreamDestroy(ctx->cp_out);
    cudaEventDestroy(ctx->ev_entry);
    for (int c = 0; c < pd_ctx::kMaxChunks; ++c) {
      cudaEventDestroy(ctx->ev_in[c]);
      cudaEventDestroy(ctx->ev_out[c]);
    }
  }
  if (ctx->host_status) cudaFreeHost(ctx->host_status);
  if (ctx->h_flag) cudaFreeHost(ctx->h_flag);
  ctx->d_flag.release();
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

const char* pd_last_error(const pd_ctx* ctx) { return ctx ? ctx->last_error.c_str() : "null context"; }

pd_status pd_set_stream(pd_ctx* ctx, void* stream) {
  if (!ctx) return PD_INVALID_ARGUMENT;
  ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  return PD_OK;
}

pd_status pd_synchronize(pd_ctx* ctx) {
  if (!ctx) return PD_INVALID_ARGUMENT;
  PD_CUDA(cudaSetDevice(ctx->device));
  PD_CUDA(cudaStreamSynchronize(ctx->stream));
  return PD_OK;
}

int64_t pd_kernel_launches(const pd_ctx* ctx) { return ctx ? ctx->launches : 0; }

const char* pd_kernel_variant(const pd_ctx* ctx, pd_algo algo, int32_t n_links) {
  (void)ctx;
  switch (algo) {
    case PD_ABIA: return "abia_ring_kernel (lane per chain, 3 fused base-frame passes, persistent CTAs, TMA producer "
                         "warp + per-pass byte ring); abia_cta_kernel for n >= 64 in batches <= 2 x SMs (CTA per chain)";
    case PD_CFA: return n_links <= 128 ? "cfa_row_kernel (CTA per chain, thread per row, row blocks in registers, OEE "
                                        "in smem); tau_surplus_lane_kernel pre-pass for batches >= 128 x SMs"
                 : n_links <= 256 ? "cfa_ws_kernel for 2 x SMs <= batch < 128 x SMs (persistent, warp-specialised: OEE "
                                    "rows of chain k beside the kinematics / tau_delta of chain k+1); otherwise "
                                    "cfa_row_kernel (CTA per chain, thread per row, OEE in smem), tau_surplus_lane_kernel "
                                    "pre-pass for batches >= 128 x SMs"
                 : cfa_workspace_bytes(n_links) <= 220 * 1024 ? "cfa_cta_kernel<smem> (CTA per chain, OEE in smem)"
                                                                    : "cfa_cta_kernel<global> (CTA per chain, L2 workspace); batches "
                                                                      "<= 4: CTA prologue + grid-wide cooperative OEE (cfa_oee_coop)";
    case PD_JSIIA: return n_links <= 64 ? "jsiia_dmma_kernel (warp per chain, M and blocked Cholesky on FP64 tensor cores, DMMA 8x8x4)"
                          : jsiia_smem_path(n_links)
                              ? "jsiia_tiled_kernel<smem> (CTA per chain, CRBA scans + 32x32-tile Cholesky in smem)"
                              : "jsiia_tiled_kernel<global> (CTA per chain, 32x32-tile Cholesky, L2 workspace); batches "
                                "<= 4: CTA build + grid-wide cooperative tile Cholesky (jsiia_factor_coop) + CTA solve";
  }
  return "unknown";
}

pd_status pd_set_models(pd_ctx* ctx, int64_t n_models, int32_t n_links, const double* links, const double* gravity,
                        int32_t* model_status, int32_t* model_rule) {
  if (!ctx) return PD_INVALID_ARGUMENT;
  if (n_models <= 0 || n_links <= 0 || !links) {
    ctx->last_error = "forward dynamics: chain has no links";
    return PD_INVALID_ARGUMENT;
  }
  PD_CUDA(cudaSetDevice(ctx->device));
  std::vector<double> g(3 * n_models);
  for (int64_t m = 0; m < n_models; ++m)
    for (int k = 0; k < 3; ++k) g[3 * m + k] = gravity ? gravity[3 * m + k] : (k == 2 ? -9.81 : 0.0);
  const size_t raw_bytes = sizeof(double) * PD_LINK_FIELDS * n_links * (size_t)n_models;
  if (ctx->models_cached && ctx->n_models == n_models && ctx->n_links == n_links && ctx->last_grav == g &&
      std::memcmp(ctx->last_links.data(), links, raw_bytes) == 0) {
    if (model_status) std::memcpy(model_status, ctx->h_mstatus.data(), sizeof(int32_t) * n_models);
    if (model_rule) std::memcpy(model_rule, ctx->h_mrule.data(), sizeof(int32_t) * n_models);
    return PD_OK;
  }
  ctx->models_cached = false;
  PD_CUDA(ctx->raw.ensure(raw_bytes + sizeof(double) * 3 * n_models));
  const int64_t model_ld = (n_models + 31) / 32 * 32;
  PD_CUDA(ctx->model.ensure(sizeof(double) * F_COUNT * n_links * (size_t)model_ld));
  PD_CUDA(ctx->gravity.ensure(sizeof(double) * 3 * n_models));
  PD_CUDA(ctx->mstatus.ensure(sizeof(int32_t) * n_models));
  PD_CUDA(ctx->mrule.ensure(sizeof(int32_t) * n_models));
  double* raw = ctx->raw.as<double>();
  double* graw = raw + PD_LINK_FIELDS * n_links * (size_t)n_models;
  PD_CUDA(cudaMemcpyAsync(raw, links, raw_bytes, cudaMemcpyHostToDevice, ctx->stream));
  PD_CUDA(cudaMemcpyAsync(graw, g.data(), sizeof(double) * 3 * n_models, cudaMemcpyHostToDevice, ctx->stream));
  // spatial_inertia_from's rules for every link, on the device (one thread per
  // model, the same arithmetic as the host link_rule; 67M links of a c5 model
  // set would take seconds on one host thread)
  launch_validate_models(raw, n_links, n_models, ctx->mstatus.as<int32_t>(), ctx->mrule.as<int32_t>(), ctx->stream);
  ctx->h_mstatus.assign(n_models, 0);
  ctx->h_mrule.assign(n_models, 0);
  PD_CUDA(cudaMemcpyAsync(ctx->h_mstatus.data(), ctx->mstatus.p, sizeof(int32_t) * n_models, cudaMemcpyDeviceToHost,
                          ctx->stream));
  PD_CUDA(cudaMemcpyAsync(ctx->h_mrule.data(), ctx->mrule.p, sizeof(int32_t) * n_models, cudaMemcpyDeviceToHost,
                          ctx->stream));
  dim3 grid((unsigned)((n_models + 127) / 128), (unsigned)n_links);
  pack_models_kernel<<<grid, 128, 0, ctx->stream>>>(raw, graw, n_links, n_models, model_ld,
                                                     ctx->model.as<double>(), ctx->gravity.as<double>());
  ctx->launches += 3;
  PD_CUDA(cudaGetLastError());
  PD_CUDA(cudaStreamSynchronize(ctx->stream));
  if (model_status) std::memcpy(model_status, ctx->h_mstatus.data(), sizeof(int32_t) * n_models);
  if (model_rule) std::memcpy(model_rule, ctx->h_mrule.data(), sizeof(int32_t) * n_models);
  ctx->n_links = n_links;
  ctx->n_models = n_models;
  ctx->model_ld = model_ld;
  ctx->model_cl_valid = false;
  // keep a copy for the identical-model check only for small model sets (a
  // chain re-sent with every single-problem call); a batch's slices are not
  // worth a host copy
  if (n_models <= 1024 && raw_bytes <= ((size_t)64 << 20)) {
    ctx->last_links.assign(links, links + raw_bytes / sizeof(double));
    ctx->last_grav = g;
    ctx->models_cached = true;
  }
  return PD_OK;
}

pd_status pd_forward_dynamics_device(pd_ctx* ctx, pd_algo algo, int64_t batch, const double* d_q,
                                     const double* d_qdot, const double* d_tau, double* d_qddot,
                                     int32_t* d_slot_status, int32_t* d_slot_round, int32_t* d_slot_index) {
  if (!ctx) return PD_INVALID_ARGUMENT;
  if (batch < 0) {
    ctx->last_error = "forward dynamics: negative batch";
    return PD_INVALID_ARGUMENT;
  }
  PD_CUDA(cudaSetDevice(ctx->device));
  if (ctx->n_models > 1 && ctx->n_models != batch) {
    ctx->last_error = "forward dynamics: batch must equal the number of models (or use one shared model)";
    return PD_INVALID_ARGUMENT;
  }
  return run_device(ctx, algo, batch, batch, d_q, d_qdot, d_tau, d_qddot, d_slot_status, d_slot_round,
                    d_slot_index);
}

}  // extern "C"

namespace {

// Host buffers [problem][link] in and out through a chunked pipeline: the
// copy-in stream streams chunk c+1 over PCIe while the compute stream
// transposes and solves chunk c and the copy-out stream returns chunk c-1.
// Chunks are 32-aligned (TMA bases stay 16-byte aligned); every chunk selects
// its kernels for the whole batch, so the results are those of the device
// path on the same problems.
pd_status host_forward_dynamics(pd_ctx* ctx, pd_algo algo, int64_t batch, const double* q, const double* qdot,
                                const double* tau, double* qddot, int32_t* slot_status, int32_t* slot_round,
                                int32_t* slot_index, Route route) {
  if (!ctx) return PD_INVALID_ARGUMENT;
  if (batch < 0 || (batch > 0 && (!q || !qdot || !tau || !qddot))) {
    ctx->last_error = "forward dynamics: null buffer";
    return PD_INVALID_ARGUMENT;
  }
  if (batch == 0) return PD_OK;
  PD_CUDA(cudaSetDevice(ctx->device));
  if (ctx->n_models <= 0 || ctx->n_links <= 0) {
    ctx->last_error = "forward dynamics: no models set (pd_set_models)";
    return PD_INVALID_ARGUMENT;
  }
  if (ctx->n_models != 1 && ctx->n_models != batch) {
    ctx->last_error = "forward dynamics: batch must equal the number of models (or use one shared model)";
    return PD_INVALID_ARGUMENT;
  }
  const int n = ctx->n_links;
  const int64_t lds = (batch + 31) / 32 * 32;  // padded link stride (TMA-friendly)
  const size_t half = (size_t)n * lds;
  // staging: [B][n] host rows -> device rows (upper half) -> [n][lds] (lower half)
  PD_CUDA(ctx->io_q.ensure(2 * sizeof(double) * half));
  PD_CUDA(ctx->io_qd.ensure(2 * sizeof(double) * half));
  PD_CUDA(ctx->io_tau.ensure(2 * sizeof(double) * half));
  PD_CUDA(ctx->io_qdd.ensure(2 * sizeof(double) * half));
  PD_CUDA(ctx->io_status.ensure(sizeof(int32_t) * 3 * batch));
  if (!ctx->cp_in) {
    PD_CUDA(cudaStreamCreateWithFlags(&ctx->cp_in, cudaStreamNonBlocking));
    PD_CUDA(cudaStreamCreateWithFlags(&ctx->cp_out, cudaStreamNonBlocking));
    PD_CUDA(cudaEventCreateWithFlags(&ctx->ev_entry, cudaEventDisableTiming));
    for (int c = 0; c < pd_ctx::kMaxChunks; ++c) {
      PD_CUDA(cudaEventCreateWithFlags(&ctx->ev_in[c], cudaEventDisableTiming));
      PD_CUDA(cudaEventCreateWithFlags(&ctx->ev_out[c], cudaEventDisableTiming));
    }
  }
  double* sq = ctx->io_q.as<double>();
  double* sqd = ctx->io_qd.as<double>();
  double* stau = ctx->io_tau.as<double>();
  double* sqdd = ctx->io_qdd.as<double>();
  int32_t* st = ctx->io_status.as<int32_t>();
  // ~8K problems per chunk, at most 8 chunks: smaller chunks add per-chunk
  // launch / event overhead faster than they shorten the pipeline's tail
  // (tools/e2e_probe.py: c2 1.50 ms at 16 chunks, 1.35 ms at 8)
  const int nch = (int)std::min<int64_t>(8, std::max<int64_t>(1, batch / 8192));
  const int64_t csz = ((batch + nch - 1) / nch + 31) / 32 * 32;
  const int64_t selB = ctx->selection_batch > 0 ? ctx->selection_batch : batch;
  PD_CUDA(cudaEventRecord(ctx->ev_entry, ctx->stream));  // earlier work on the staging buffers
  PD_CUDA(cudaStreamWaitEvent(ctx->cp_in, ctx->ev_entry, 0));
  PD_CUDA(cudaStreamWaitEvent(ctx->cp_out, ctx->ev_entry, 0));
  std::string variant;
  for (int c = 0; c < nch; ++c) {
    const int64_t b0 = c * csz, nb = std::min<int64_t>(csz, batch - b0);
    if (nb <= 0) break;
    const size_t off = (size_t)b0 * n, bytes = sizeof(double) * (size_t)n * nb;
    PD_CUDA(cudaMemcpyAsync(sq + half + off, q + off, bytes, cudaMemcpyHostToDevice, ctx->cp_in));
    PD_CUDA(cudaMemcpyAsync(sqd + half + off, qdot + off, bytes, cudaMemcpyHostToDevice, ctx->cp_in));
    PD_CUDA(cudaMemcpyAsync(stau + half + off, tau + off, bytes, cudaMemcpyHostToDevice, ctx->cp_in));
    PD_CUDA(cudaEventRecord(ctx->ev_in[c], ctx->cp_in));
    PD_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_in[c], 0));
    launch_transpose3(ctx, sq + half + off, sqd + half + off, stau + half + off, sq + b0, sqd + b0, stau + b0, nb, n,
                      n, lds);
    pd_status s = run_device(ctx, algo, nb, lds, sq + b0, sqd + b0, stau + b0, sqdd + b0, st + b0, st + batch + b0,
                             st + 2 * batch + b0, b0, selB, route);
    if (s != PD_OK) return s;
    if (c == 0) variant = ctx->last_variant;
    launch_transpose(ctx, sqdd + b0, sqdd + half + off, n, nb, lds, n);
    PD_CUDA(cudaEventRecord(ctx->ev_out[c], ctx->stream));
    PD_CUDA(cudaStreamWaitEvent(ctx->cp_out, ctx->ev_out[c], 0));
    PD_CUDA(cudaMemcpyAsync(qddot + off, sqdd + half + off, bytes, cudaMemcpyDeviceToHost, ctx->cp_out));
  }
  if (nch > 1) ctx->last_variant = variant + " x " + std::to_string(nch) + " chunks";
  const bool want_status = slot_status || slot_round || slot_index;
  if (!want_status) {
    PD_CUDA(cudaStreamSynchronize(ctx->cp_out));
    PD_CUDA(cudaStreamSynchronize(ctx->stream));
    return PD_OK;
  }
  // Slot outcomes: one device-side OR over the statuses; when every slot
  // succeeded (round and index are then 0 too) the host arrays are zero-
  // filled instead of copying 12 bytes per problem back over PCIe.
  if (!ctx->h_flag) PD_CUDA(cudaMallocHost(&ctx->h_flag, sizeof(int32_t)));
  PD_CUDA(ctx->d_flag.ensure(sizeof(int32_t)));
  PD_CUDA(cudaMemsetAsync(ctx->d_flag.p, 0, sizeof(int32_t), ctx->stream));
  any_status_kernel<<<(unsigned)std::min<int64_t>((batch + 255) / 256, 1024), 256, 0, ctx->stream>>>(
      st, batch, ctx->d_flag.as<int32_t>());
  ctx->launches++;
  PD_CUDA(cudaMemcpyAsync(ctx->h_flag, ctx->d_flag.p, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
  PD_CUDA(cudaStreamSynchronize(ctx->stream));
  if (*ctx->h_flag == 0) {
    PD_CUDA(cudaStreamSynchronize(ctx->cp_out));
    if (slot_status) std::memset(slot_status, 0, sizeof(int32_t) * batch);
    if (slot_round) std::memset(slot_round, 0, sizeof(int32_t) * batch);
    if (slot_index) std::memset(slot_index, 0, sizeof(int32_t) * batch);
    return PD_OK;
  }
  if (ctx->host_status_n < (size_t)(3 * batch)) {
    if (ctx->host_status) cudaFreeHost(ctx->host_status);
    ctx->host_status = nullptr;
    ctx->host_status_n = 0;
    PD_CUDA(cudaMallocHost(&ctx->host_status, sizeof(int32_t) * 3 * batch));
    ctx->host_status_n = (size_t)(3 * batch);
  }
  PD_CUDA(cudaMemcpyAsync(ctx->host_status, st, sizeof(int32_t) * 3 * batch, cudaMemcpyDeviceToHost, ctx->cp_out));
  PD_CUDA(cudaStreamSynchronize(ctx->cp_out));
  const int32_t* hs = ctx->host_status;
  if (slot_status) std::memcpy(slot_status, hs, sizeof(int32_t) * batch);
  if (slot_round) std::memcpy(slot_round, hs + batch, sizeof(int32_t) * batch);
  if (slot_index) std::memcpy(slot_index, hs + 2 * batch, sizeof(int32_t) * batch);
  return PD_OK;
}

}  // namespace

extern "C" {

pd_status pd_forward_dynamics(pd_ctx* ctx, pd_algo algo, int64_t batch, const double* q, const double* qdot,
                              const double* tau, double* qddot, int32_t* slot_status, int32_t* slot_round,
                              int32_t* slot_index) {
  return host_forward_dynamics(ctx, algo, batch, q, qdot, tau, qddot, slot_status, slot_round, slot_index,
                               ROUTE_AUTO);
}

pd_status pd_forward_dynamics_traced(pd_ctx* ctx, pd_algo algo, int64_t batch, const double* q, const double* qdot,
                                     const double* tau, double* qddot, int32_t* slot_status, int32_t* slot_round,
                                     int32_t* slot_index, pd_exec_trace* trace) {
  pd_status s = host_forward_dynamics(ctx, algo, batch, q, qdot, tau, qddot, slot_status, slot_round, slot_index,
                                      ROUTE_LOG_DEPTH);
  if (s == PD_OK && trace && batch > 0) *trace = ctx->last_trace;
  return s;
}

const char* pd_last_variant(const pd_ctx* ctx) { return ctx ? ctx->last_variant.c_str() : ""; }

pd_status pd_last_trace(const pd_ctx* ctx, pd_exec_trace* trace) {
  if (!ctx || !trace) return PD_INVALID_ARGUMENT;
  *trace = ctx->last_trace;
  return PD_OK;
}

pd_status pd_set_selection_batch(pd_ctx* ctx, int64_t batch) {
  if (!ctx || batch < 0) return PD_INVALID_ARGUMENT;
  ctx->selection_batch = batch;
  return PD_OK;
}

}  // extern "C"

namespace {

IdOpts id_opts(const pd_id_options* o) {
  IdOpts r{};
  r.gravity = 1;
  if (o) {
    for (int k = 0; k < 6; ++k) {
      r.bv[k] = o->base_velocity[k];
      r.ba[k] = o->base_acceleration[k];
      r.tip[k] = o->tip_wrench[k];
    }
    r.gravity = o->apply_gravity != 0;
  }
  return r;
}

// Reference behaviour for a bad model in the single-chain ID / JSI calls:
// link_inertias -> spatial_inertia_from throws std::invalid_argument
// (model.cpp:148-155, spatial.cpp:72-87).
pd_status check_models(pd_ctx* ctx, int64_t batch, const char* what) {
  if (ctx->n_models <= 0 || (ctx->n_models != 1 && ctx->n_models != batch)) {
    ctx->last_error = std::string(what) + ": batch must equal the number of models (or use one shared model)";
    return PD_INVALID_ARGUMENT;
  }
  const int64_t m_end = ctx->n_models == 1 ? 1 : batch;
  for (int64_t m = 0; m < m_end && m < (int64_t)ctx->h_mstatus.size(); ++m)
    if (ctx->h_mstatus[m] != PD_SLOT_OK) {
      char buf[256];
      pd_slot_message(ctx->h_mstatus[m], 0, ctx->h_mrule[m], ctx->n_links, buf, sizeof buf);
      ctx->last_error = buf;
      return PD_INVALID_ARGUMENT;
    }
  return PD_OK;
}

// Host-buffer inverse dynamics: [problem][link] in, [problem][link] out;
// link states (nullable) [problem][link][6].
pd_status run_idyn_host(pd_ctx* ctx, int64_t batch, const double* q, const double* qdot, const double* qddot,
                        const pd_id_options* opts, double* tau, double* vel, double* acc, double* frc) {
  if (!ctx) return PD_INVALID_ARGUMENT;
  if (batch < 0 || (batch > 0 && (!q || !qdot))) {
    ctx->last_error = "inverse dynamics: null buffer";
    return PD_INVALID_ARGUMENT;
  }
  if (batch == 0) return PD_OK;
  pd_status cs = check_models(ctx, batch, "inverse dynamics");
  if (cs != PD_OK) return cs;
  PD_CUDA(cudaSetDevice(ctx->device));
  const int n = ctx->n_links;
  const size_t bytes = sizeof(double) * (size_t)n * batch;
  const size_t half = (size_t)n * batch;
  const bool states = vel || acc || frc;
  PD_CUDA(ctx->io_q.ensure(2 * bytes));
  PD_CUDA(ctx->io_qd.ensure(2 * bytes));
  PD_CUDA(ctx->io_tau.ensure(2 * bytes));
  PD_CUDA(ctx->io_qdd.ensure(2 * bytes));
  PD_CUDA(ctx->io_status.ensure(sizeof(int32_t) * 3 * batch));
  if (states) PD_CUDA(ctx->states.ensure(2 * 3 * 6 * bytes));
  double *sq = ctx->io_q.as<double>(), *sqd = ctx->io_qd.as<double>(), *sqdd = ctx->io_qdd.as<double>(),
         *stau = ctx->io_tau.as<double>();
  PD_CUDA(cudaMemcpyAsync(sq + half, q, bytes, cudaMemcpyHostToDevice, ctx->stream));
  PD_CUDA(cudaMemcpyAsync(sqd + half, qdot, bytes, cudaMemcpyHostToDevice, ctx->stream));
  if (qddot)
    PD_CUDA(cudaMemcpyAsync(sqdd + half, qddot, bytes, cudaMemcpyHostToDevice, ctx->stream));
  else
    PD_CUDA(cudaMemsetAsync(sqdd, 0, bytes, ctx->stream));
  launch_transpose(ctx, sq + half, sq, batch, n, n, batch);
  launch_transpose(ctx, sqd + half, sqd, batch, n, n, batch);
  if (qddot) launch_transpose(ctx, sqdd + half, sqdd, batch, n, n, batch);
  int32_t* st = ctx->io_status.as<int32_t>();
  double* sv = states ? ctx->states.as<double>() : nullptr;  // 3 x [n][6][batch], then 3 x host-order staging
  const size_t sn = 6 * half;
  // BatchIO: tau slot carries qddot in, qdd slot carries torques out
  BatchIO io{sq, sqd, sqdd, stau, st, st + batch, st + 2 * batch, batch, batch};
  launch_idyn(model_view(ctx), io, id_opts(opts), ctx->raw.as<double>(), sv, sv ? sv + sn : nullptr,
              sv ? sv + 2 * sn : nullptr, ctx->stream);
  ctx->launches++;
  // lane per chain: the V / A and F recursions walk the n links sequentially
  note_variant(ctx, "idyn_lane_kernel", 0, n, 0, 0);
  PD_CUDA(cudaGetLastError());
  if (tau) {
    launch_transpose(ctx, stau, stau + half, n, batch, batch, n);
    PD_CUDA(cudaMemcpyAsync(tau, stau + half, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  }
  double* outs[3] = {vel, acc, frc};
  for (int k = 0; k < 3; ++k)
    if (outs[k]) {
      // [link][6][problem] -> [problem][link][6]
      launch_transpose(ctx, sv + k * sn, sv + (3 + k) * sn, 6 * (int64_t)n, batch, batch, 6 * (int64_t)n);
      PD_CUDA(cudaMemcpyAsync(outs[k], sv + (3 + k) * sn, 6 * bytes, cudaMemcpyDeviceToHost, ctx->stream));
    }
  PD_CUDA(cudaStreamSynchronize(ctx->stream));
  return PD_OK;
}

}  // namespace

extern "C" {

pd_status pd_inverse_dynamics(pd_ctx* ctx, int64_t batch, const double* q, const double* qdot, const double* qddot,
                              double* tau) {
  if (ctx && batch > 0 && (!qddot || !tau)) {
    ctx->last_error = "inverse dynamics: null buffer";
    return PD_INVALID_ARGUMENT;
  }
  return run_idyn_host(ctx, batch, q, qdot, qddot, nullptr, tau, nullptr, nullptr, nullptr);
}

pd_status pd_inverse_dynamics_opts(pd_ctx* ctx, int64_t batch, const double* q, const double* qdot,
                                   const double* qddot, const pd_id_options* opts, double* tau) {
  if (ctx && batch > 0 && (!qddot || !tau)) {
    ctx->last_error = "inverse dynamics: null buffer";
    return PD_INVALID_ARGUMENT;
  }
  return run_idyn_host(ctx, batch, q, qdot, qddot, opts, tau, nullptr, nullptr, nullptr);
}

pd_status pd_bias_torque(pd_ctx* ctx, int64_t batch, const double* q, const double* qdot, double* tau) {
  if (ctx && batch > 0 && !tau) {
    ctx->last_error = "inverse dynamics: null buffer";
    return PD_INVALID_ARGUMENT;
  }
  return run_idyn_host(ctx, batch, q, qdot, nullptr, nullptr, tau, nullptr, nullptr, nullptr);
}

pd_status pd_link_states(pd_ctx* ctx, int64_t batch, const double* q, const double* qdot, const double* qddot,
                         const pd_id_options* opts, double* velocity, double* acceleration, double* force) {
  if (ctx && batch > 0 && (!qddot || !velocity || !acceleration || !force)) {
    ctx->last_error = "link states: null buffer";
    return PD_INVALID_ARGUMENT;
  }
  return run_idyn_host(ctx, batch, q, qdot, qddot, opts, nullptr, velocity, acceleration, force);
}

pd_status pd_inverse_dynamics_device(pd_ctx* ctx, int64_t batch, const double* d_q, const double* d_qdot,
                                     const double* d_qddot, const pd_id_options* opts, double* d_tau) {
  if (!ctx) return PD_INVALID_ARGUMENT;
  if (batch < 0 || (batch > 0 && (!d_q || !d_qdot || !d_qddot || !d_tau))) {
    ctx->last_error = "inverse dynamics: null buffer";
    return PD_INVALID_ARGUMENT;
  }
  if (batch == 0) return PD_OK;
  pd_status cs = check_models(ctx, batch, "inverse dynamics");
  if (cs != PD_OK) return cs;
  PD_CUDA(cudaSetDevice(ctx->device));
  PD_CUDA(ctx->io_status.ensure(sizeof(int32_t) * 3 * batch));
  int32_t* st = ctx->io_status.as<int32_t>();
  BatchIO io{d_q, d_qdot, d_qddot, d_tau, st, st + batch, st + 2 * batch, batch, batch};
  launch_idyn(model_view(ctx), io, id_opts(opts), ctx->raw.as<double>(), nullptr, nullptr, nullptr, ctx->stream);
  ctx->launches++;
  note_variant(ctx, "idyn_lane_kernel", 0, ctx->n_links, 0, 0);
  PD_CUDA(cudaGetLastError());
  return PD_OK;
}

pd_status pd_joint_space_inertia(pd_ctx* ctx, int64_t batch, const double* q, double* M) {
  if (!ctx) return PD_INVALID_ARGUMENT;
  if (batch < 0 || (batch > 0 && (!q || !M))) {
    ctx->last_error = "joint_space_inertia: null buffer";
    return PD_INVALID_ARGUMENT;
  }
  if (batch == 0) return PD_OK;
  pd_status cs = check_models(ctx, batch, "joint_space_inertia");
  if (cs != PD_OK) return cs;
  PD_CUDA(cudaSetDevice(ctx->device));
  const int n = ctx->n_links;
  const size_t bytes = sizeof(double) * (size_t)n * batch;
  const size_t mbytes = sizeof(double) * (size_t)n * n * batch;
  PD_CUDA(ctx->io_q.ensure(2 * bytes));
  PD_CUDA(ctx->io_qdd.ensure(mbytes));
  PD_CUDA(ctx->io_status.ensure(sizeof(int32_t) * 3 * batch));
  double* sq = ctx->io_q.as<double>();
  PD_CUDA(cudaMemcpyAsync(sq + (size_t)n * batch, q, bytes, cudaMemcpyHostToDevice, ctx->stream));
  launch_transpose(ctx, sq + (size_t)n * batch, sq, batch, n, n, batch);
  PD_CUDA(ensure_model_cl(ctx));
  ModelView mv = model_view(ctx);
  mv.fcl = ctx->model_cl.as<double>();
  int64_t slots = 0;
  if (!jsiia_smem_path(n)) {
    const size_t wsb = jsiia_workspace_bytes(n);
    slots = cta_slots(ctx, wsb, batch);
    PD_CUDA(ctx->cta_ws.ensure(wsb * slots));
  }
  int32_t* st = ctx->io_status.as<int32_t>();
  BatchIO io{sq, sq, sq, nullptr, st, st + batch, st + 2 * batch, batch, batch};
  launch_jsi(mv, io, ctx->cta_ws.as<double>(), slots, ctx->sm_count, ctx->io_qdd.as<double>(), ctx->stream);
  ctx->launches += slots ? (batch + slots - 1) / slots : 1;
  {  // CTA per chain: kinematics, S0 / J0, the composite-inertia suffix scan, the M fill
    const CtaShape cs = cta_shape(n, 32 * jsiia_warps(n, batch, ctx->sm_count));
    note_variant(ctx, std::string("jsiia_tiled_kernel<") + (slots ? "global" : "smem") + ", M only>", 4,
                 cs.lpt > 1 ? cs.lpt : 0, ceil_log2_host(cs.groups), 0);
  }
  PD_CUDA(cudaGetLastError());
  PD_CUDA(cudaMemcpyAsync(M, ctx->io_qdd.p, mbytes, cudaMemcpyDeviceToHost, ctx->stream));
  PD_CUDA(cudaStreamSynchronize(ctx->stream));
  return PD_OK;
}

void pd_slot_message(int32_t code, int32_t round, int32_t index, int32_t n_links, char* buf, int32_t buflen) {
  if (!buf || buflen <= 0) return;
  std::string m;
  switch (code) {
    case PD_SLOT_OK: m = ""; break;
    case PD_SLOT_DEGENERATE_ARTICULATION:
      m = "degenerate articulation at joint " + std::to_string(index) + ": projected articulated inertia vanishes";
      break;
    case PD_SLOT_JSI_NOT_SPD:
      m = "joint-space inertia is not positive definite; the chain model is degenerate";
      break;
    case PD_SLOT_JSI_REFINE_FAILED:
      m = "joint-space inertia solve failed to reach the required residual; the inertia matrix is too "
          "ill-conditioned";
      break;
    case PD_SLOT_LINK_INERTIA_NOT_PD:
      m = "constraint-force assembly: a link inertia is not positive definite";
      break;
    case PD_SLOT_OEE_SINGULAR_PIVOT:
      m = "odd-even elimination: singular pivot block (round " + std::to_string(round) + ", block " +
          std::to_string(index) + ")";
      break;
    case PD_SLOT_OEE_SINGULAR_FINAL:
      m = "odd-even elimination: singular diagonal block after elimination (block " + std::to_string(index) + ")";
      break;
    case PD_SLOT_BAD_MODEL:
      switch (index) {
        case PD_RULE_MASS: m = "spatial inertia: mass must be positive"; break;
        case PD_RULE_FINITE: m = "spatial inertia: parameters must be finite"; break;
        case PD_RULE_SYMMETRIC: m = "spatial inertia: rotational inertia must be symmetric"; break;
        default: m = "spatial inertia: rotational inertia must be positive definite"; break;
      }
      break;
    case PD_SLOT_BAD_SIZE:
      m = n_links <= 0 ? "forward dynamics: chain has no links"
                       : "forward dynamics: q, qdot and tau must each have one entry per joint (chain has " +
                             std::to_string(n_links) + ")";
      break;
    default: m = "unknown slot status"; break;
  }
  std::strncpy(buf, m.c_str(), (size_t)buflen - 1);
  buf[buflen - 1] = '\0';
}

}  // extern "C"

// ---------------------------------------------------------------- device workloads
extern "C" {

pd_status pd_block_bidiag_solve(pd_ctx* ctx, int32_t dim, int64_t batch, int32_t n, int32_t upper,
                                const double* coupling, const double* rhs, double* x) {
  if (!ctx) return PD_INVALID_ARGUMENT;
  if (dim < 1 || dim > 6) {
    ctx->last_error = "block bi-diagonal solve: block size must be 1..6";
    return PD_INVALID_ARGUMENT;
  }
  if (batch < 0 || n < 0 || (batch > 0 && n > 0 && (!rhs || !x || (n > 1 && !coupling)))) {
    ctx->last_error = "block bi-diagonal solve: null buffer";
    return PD_INVALID_ARGUMENT;
  }
  if (batch == 0 || n == 0) return PD_OK;
  PD_CUDA(cudaSetDevice(ctx->device));
  const size_t nc = (size_t)batch * (n - 1) * dim * dim, nr = (size_t)batch * n * dim;
  PD_CUDA(ctx->states.ensure(sizeof(double) * (nc + 2 * nr)));
  double* c = ctx->states.as<double>();
  double* r = c + nc;
  double* xo = r + nr;
  if (nc) PD_CUDA(cudaMemcpyAsync(c, coupling, sizeof(double) * nc, cudaMemcpyHostToDevice, ctx->stream));
  PD_CUDA(cudaMemcpyAsync(r, rhs, sizeof(double) * nr, cudaMemcpyHostToDevice, ctx->stream));
  launch_bidiag(dim, c, r, xo, batch, n, upper ? 1 : 0, ctx->stream);
  ctx->launches++;
  PD_CUDA(cudaGetLastError());
  PD_CUDA(cudaMemcpyAsync(x, xo, sizeof(double) * nr, cudaMemcpyDeviceToHost, ctx->stream));
  PD_CUDA(cudaStreamSynchronize(ctx->stream));
  return PD_OK;
}

pd_status pd_block_bidiag_solve6(pd_ctx* ctx, int64_t batch, int32_t n, int32_t upper, const double* coupling,
                                 const double* rhs, double* x) {
  return pd_block_bidiag_solve(ctx, 6, batch, n, upper, coupling, rhs, x);
}

pd_status pd_block_tridiag_solve(pd_ctx* ctx, int32_t block, int32_t cols, int64_t batch, int32_t n,
                                 const double* diag, const double* upper, const double* rhs, double* x,
                                 int32_t* slot_status, int32_t* slot_round, int32_t* slot_index) {
  if (!ctx) return PD_INVALID_ARGUMENT;
  if (block < 1 || block > 6 || cols < 1 || cols > 4) {
    ctx->last_error = "block tri-diagonal solve: block size must be 1..6 and right-hand-side columns 1..4";
    return PD_INVALID_ARGUMENT;
  }
  if (batch < 0 || n < 1 || n > 256 || (batch > 0 && (!diag || !rhs || !x || (n > 1 && !upper)))) {
    ctx->last_error = "block tri-diagonal solve: need 1 <= n <= 256 rows and non-null buffers";
    return PD_INVALID_ARGUMENT;
  }
  if (batch == 0) return PD_OK;
  PD_CUDA(cudaSetDevice(ctx->device));
  const size_t bb = (size_t)block * block, bm = (size_t)block * cols;
  const size_t nd = (size_t)batch * n * bb, nu = (size_t)batch * (n - 1) * bb, nr = (size_t)batch * n * bm;
  PD_CUDA(ctx->states.ensure(sizeof(double) * (nd + nu + 2 * nr) + sizeof(int32_t) * 3 * batch));
  double* d = ctx->states.as<double>();
  double* u = d + nd;
  double* r = u + nu;
  double* xo = r + nr;
  int32_t* st = reinterpret_cast<int32_t*>(xo + nr);
  PD_CUDA(cudaMemcpyAsync(d, diag, sizeof(double) * nd, cudaMemcpyHostToDevice, ctx->stream));
  if (nu) PD_CUDA(cudaMemcpyAsync(u, upper, sizeof(double) * nu, cudaMemcpyHostToDevice, ctx->stream));
  PD_CUDA(cudaMemcpyAsync(r, rhs, sizeof(double) * nr, cudaMemcpyHostToDevice, ctx->stream));
  launch_oee_block(block, cols, d, u, r, xo, batch, n, st, st + batch, st + 2 * batch, ctx->stream);
  ctx->launches++;
  PD_CUDA(cudaGetLastError());
  PD_CUDA(cudaMemcpyAsync(x, xo, sizeof(double) * nr, cudaMemcpyDeviceToHost, ctx->stream));
  std::vector<int32_t> hs(3 * batch);
  PD_CUDA(cudaMemcpyAsync(hs.data(), st, sizeof(int32_t) * 3 * batch, cudaMemcpyDeviceToHost, ctx->stream));
  PD_CUDA(cudaStreamSynchronize(ctx->stream));
  if (slot_status) std::memcpy(slot_status, hs.data(), sizeof(int32_t) * batch);
  if (slot_round) std::memcpy(slot_round, hs.data() + batch, sizeof(int32_t) * batch);
  if (slot_index) std::memcpy(slot_index, hs.data() + 2 * batch, sizeof(int32_t) * batch);
  return PD_OK;
}

pd_status pd_oee_eliminate_rounds(pd_ctx* ctx, int32_t block, int32_t cols, int64_t batch, int32_t n,
                                  int32_t distance, int32_t state_round, int32_t rounds, const double* diag,
                                  const double* coupling, const double* rhs, double* diag_out,
                                  double* coupling_out, double* rhs_out, int32_t* slot_status, int32_t* slot_round,
                                  int32_t* slot_index) {
  if (!ctx) return PD_INVALID_ARGUMENT;
  if (block < 1 || block > 6 || cols < 1 || cols > 4 || n < 1 || n > 256 || distance < 1 || state_round < 0 ||
      rounds < 0 || rounds > 30) {
    ctx->last_error = "odd-even elimination rounds: block 1..6, cols 1..4, 1 <= n <= 256, distance >= 1";
    return PD_INVALID_ARGUMENT;
  }
  const int64_t nu0 = n > distance ? n - distance : 0;
  int64_t hend = distance;
  for (int r = 0; r < rounds && hend < (1ll << 40); ++r) hend *= 2;
  const int64_t nu1 = n > hend ? n - hend : 0;
  if (batch < 0 || (batch > 0 && (!diag || !rhs || !diag_out || !rhs_out || (nu0 > 0 && !coupling) ||
                                   (nu1 > 0 && !coupling_out)))) {
    ctx->last_error = "odd-even elimination rounds: null buffer";
    return PD_INVALID_ARGUMENT;
  }
  if (batch == 0) return PD_OK;
  PD_CUDA(cudaSetDevice(ctx->device));
  const size_t bb = (size_t)block * block, bm = (size_t)block * cols;
  const size_t nd = (size_t)batch * n * bb, nc0 = (size_t)batch * nu0 * bb, nc1 = (size_t)batch * nu1 * bb,
               nr = (size_t)batch * n * bm;
  PD_CUDA(ctx->states.ensure(sizeof(double) * (2 * nd + nc0 + nc1 + 2 * nr) + sizeof(int32_t) * 3 * batch));
  double* d = ctx->states.as<double>();
  double* c = d + nd;
  double* r = c + nc0;
  double* dout = r + nr;
  double* cout = dout + nd;
  double* rout = cout + nc1;
  int32_t* st = reinterpret_cast<int32_t*>(rout + nr);
  PD_CUDA(cudaMemcpyAsync(d, diag, sizeof(double) * nd, cudaMemcpyHostToDevice, ctx->stream));
  if (nc0) PD_CUDA(cudaMemcpyAsync(c, coupling, sizeof(double) * nc0, cudaMemcpyHostToDevice, ctx->stream));
  PD_CUDA(cudaMemcpyAsync(r, rhs, sizeof(double) * nr, cudaMemcpyHostToDevice, ctx->stream));
  launch_oee_rounds(block, cols, d, c, r, batch, n, distance, state_round, rounds, dout, cout, rout, st, st + batch,
                    st + 2 * batch, ctx->stream);
  ctx->launches++;
  PD_CUDA(cudaGetLastError());
  std::vector<int32_t> hs(3 * batch);
  PD_CUDA(cudaMemcpyAsync(hs.data(), st, sizeof(int32_t) * 3 * batch, cudaMemcpyDeviceToHost, ctx->stream));
  PD_CUDA(cudaMemcpyAsync(diag_out, dout, sizeof(double) * nd, cudaMemcpyDeviceToHost, ctx->stream));
  if (nc1) PD_CUDA(cudaMemcpyAsync(coupling_out, cout, sizeof(double) * nc1, cudaMemcpyDeviceToHost, ctx->stream));
  PD_CUDA(cudaMemcpyAsync(rhs_out, rout, sizeof(double) * nr, cudaMemcpyDeviceToHost, ctx->stream));
  PD_CUDA(cudaStreamSynchronize(ctx->stream));
  if (slot_status) std::memcpy(slot_status, hs.data(), sizeof(int32_t) * batch);
  if (slot_round) std::memcpy(slot_round, hs.data() + batch, sizeof(int32_t) * batch);
  if (slot_index) std::memcpy(slot_index, hs.data() + 2 * batch, sizeof(int32_t) * batch);
  return PD_OK;
}

pd_status pd_block_tridiag_solve5(pd_ctx* ctx, int64_t batch, int32_t n, const double* diag, const double* upper,
                                  const double* rhs, double* x, int32_t* slot_status, int32_t* slot_round,
                                  int32_t* slot_index) {
  return pd_block_tridiag_solve(ctx, 5, 1, batch, n, diag, upper, rhs, x, slot_status, slot_round, slot_index);
}

pd_status pd_workload_chains_device(pd_ctx* ctx, uint64_t cell_seed, int32_t n_links, int64_t g0, int64_t count,
                                    double* d_links) {
  if (!ctx) return PD_INVALID_ARGUMENT;
  if (n_links <= 0 || count < 0 || g0 < 0 || (count > 0 && !d_links)) {
    ctx->last_error = "workload chains: invalid arguments";
    return PD_INVALID_ARGUMENT;
  }
  if (count == 0) return PD_OK;
  PD_CUDA(cudaSetDevice(ctx->device));
  launch_workload_chains(cell_seed, n_links, g0, count, d_links, ctx->stream);
  ctx->launches++;
  PD_CUDA(cudaGetLastError());
  return PD_OK;
}

pd_status pd_set_models_workload(pd_ctx* ctx, uint64_t cell_seed, int32_t n_links, int64_t g0, int64_t count,
                                 const double* gravity, int32_t* model_status, int32_t* model_rule) {
  if (!ctx) return PD_INVALID_ARGUMENT;
  if (count <= 0 || n_links <= 0 || g0 < 0) {
    ctx->last_error = "forward dynamics: chain has no links";
    return PD_INVALID_ARGUMENT;
  }
  PD_CUDA(cudaSetDevice(ctx->device));
  ctx->models_cached = false;
  const int64_t n_models = count;
  const size_t raw_bytes = sizeof(double) * PD_LINK_FIELDS * n_links * (size_t)n_models;
  PD_CUDA(ctx->raw.ensure(raw_bytes + sizeof(double) * 3 * n_models));
  const int64_t model_ld = (n_models + 31) / 32 * 32;
  PD_CUDA(ctx->model.ensure(sizeof(double) * F_COUNT * n_links * (size_t)model_ld));
  PD_CUDA(ctx->gravity.ensure(sizeof(double) * 3 * n_models));
  PD_CUDA(ctx->mstatus.ensure(sizeof(int32_t) * n_models));
  PD_CUDA(ctx->mrule.ensure(sizeof(int32_t) * n_models));
  double* raw = ctx->raw.as<double>();
  double* graw = raw + PD_LINK_FIELDS * n_links * (size_t)n_models;
  launch_workload_chains(cell_seed, n_links, g0, count, raw, ctx->stream);
  std::vector<double> g(3 * n_models);
  for (int64_t m = 0; m < n_models; ++m)
    for (int k = 0; k < 3; ++k) g[3 * m + k] = gravity ? gravity[k] : (k == 2 ? -9.81 : 0.0);
  PD_CUDA(cudaMemcpyAsync(graw, g.data(), sizeof(double) * 3 * n_models, cudaMemcpyHostToDevice, ctx->stream));
  launch_validate_models(raw, n_links, n_models, ctx->mstatus.as<int32_t>(), ctx->mrule.as<int32_t>(), ctx->stream);
  ctx->h_mstatus.assign(n_models, 0);
  ctx->h_mrule.assign(n_models, 0);
  PD_CUDA(cudaMemcpyAsync(ctx->h_mstatus.data(), ctx->mstatus.p, sizeof(int32_t) * n_models, cudaMemcpyDeviceToHost,
                          ctx->stream));
  PD_CUDA(cudaMemcpyAsync(ctx->h_mrule.data(), ctx->mrule.p, sizeof(int32_t) * n_models, cudaMemcpyDeviceToHost,
                          ctx->stream));
  dim3 grid((unsigned)((n_models + 127) / 128), (unsigned)n_links);
  pack_models_kernel<<<grid, 128, 0, ctx->stream>>>(raw, graw, n_links, n_models, model_ld, ctx->model.as<double>(),
                                                     ctx->gravity.as<double>());
  ctx->launches += 4;
  ctx->models_cached = false;
  PD_CUDA(cudaGetLastError());
  PD_CUDA(cudaStreamSynchronize(ctx->stream));
  if (model_status) std::memcpy(model_status, ctx->h_mstatus.data(), sizeof(int32_t) * n_models);
  if (model_rule) std::memcpy(model_rule, ctx->h_mrule.data(), sizeof(int32_t) * n_models);
  ctx->n_links = n_links;
  ctx->n_models = n_models;
  ctx->model_ld = model_ld;
  ctx->model_cl_valid = false;
  return PD_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- operator builders (operators.cu)
namespace pd {
void launch_kinematics(const double* raw, int n, int64_t n_models, int64_t batch, const double* q, double* rel,
                       double* base_transport, double* transport, double* screw, cudaStream_t s);
void launch_link_inertias(const double* raw, int64_t count, double* out, cudaStream_t s);
void launch_abi(int64_t batch, int n, const double* transport, const double* inertia, int64_t inertia_stride,
                const double* screw, double* abi, double* joint_inertia, double* gain, int32_t* status,
                int32_t* index, cudaStream_t s);
void launch_basis(int64_t count, const double* screw, double* basis, cudaStream_t s);
void launch_cfa_ops(int64_t batch, int n, const double* inertia, int64_t istride, const double* transport,
                    const double* screw, const double* basis, double* diag, double* upper, double* cross_sub,
                    double* cross_diag, double* cross_super, double* joint_diag, double* joint_off, int32_t* bad_link,
                    cudaStream_t s);
void launch_cfa_apply(int op, int64_t batch, int n, const double* cross_sub, const double* cross_diag,
                      const double* cross_super, const double* joint_diag, const double* joint_off, const double* in,
                      double* out, cudaStream_t s);
void launch_propagate_setup(int kind, int64_t batch, int n, const double* base_transport, const double* transport,
                            const double* screw, const double* inertia, int64_t istride, const double* qdot,
                            const double* qddot, const double* vel, const double* acc, const double* boundary,
                            double* coupling, double* rhs, cudaStream_t s);
}  // namespace pd

namespace {

// One host-buffer call of an operator builder: inputs are copied into one
// device arena, the kernel runs, outputs come back; the arena (ctx->states)
// is reused across calls.
struct Arena {
  struct In {
    const void* host;
    size_t bytes;
  };
  struct Out {
    void* host;
    size_t bytes;
  };
  std::vector<In> ins;
  std::vector<Out> outs;
  std::vector<size_t> in_off, out_off;
  char* base = nullptr;
  size_t add_in(const void* h, size_t b) {
    ins.push_back({h, b});
    return ins.size() - 1;
  }
  size_t add_out(void* h, size_t b) {
    outs.push_back({h, b});
    return outs.size() - 1;
  }
  pd_status stage(pd_ctx* ctx) {
    size_t off = 0;
    auto pad = [](size_t b) { return (b + 255) / 256 * 256; };
    for (const In& i : ins) {
      in_off.push_back(off);
      off += pad(i.bytes);
    }
    for (const Out& o : outs) {
      out_off.push_back(off);
      off += pad(o.bytes);
    }
    PD_CUDA(ctx->states.ensure(off + 256));
    base = ctx->states.as<char>();
    for (size_t k = 0; k < ins.size(); ++k)
      if (ins[k].bytes)
        PD_CUDA(cudaMemcpyAsync(base + in_off[k], ins[k].host, ins[k].bytes, cudaMemcpyHostToDevice, ctx->stream));
    return PD_OK;
  }
  template <class T>
  T* in(size_t k) const {
    return reinterpret_cast<T*>(base + in_off[k]);
  }
  template <class T>
  T* out(size_t k) const {
    return reinterpret_cast<T*>(base + out_off[k]);
  }
  pd_status finish(pd_ctx* ctx) {
    PD_CUDA(cudaGetLastError());
    for (size_t k = 0; k < outs.size(); ++k)
      if (outs[k].bytes && outs[k].host)
        PD_CUDA(cudaMemcpyAsync(outs[k].host, base + out_off[k], outs[k].bytes, cudaMemcpyDeviceToHost, ctx->stream));
    PD_CUDA(cudaStreamSynchronize(ctx->stream));
    return PD_OK;
  }
};

bool bad_args(pd_ctx* ctx, bool bad, const char* what) {
  if (bad) ctx->last_error = what;
  return bad;
}

}  // namespace

extern "C" {

pd_status pd_assemble_kinematics(pd_ctx* ctx, int64_t batch, const double* q, double* rel, double* base_transport,
                                 double* transport, double* screw) {
  if (!ctx) return PD_INVALID_ARGUMENT;
  if (bad_args(ctx, batch < 0 || (batch > 0 && (!q || !rel || !base_transport || !screw)),
               "assemble_kinematics: null buffer"))
    return PD_INVALID_ARGUMENT;
  if (batch == 0) return PD_OK;
  if (ctx->n_models <= 0 || (ctx->n_models != 1 && ctx->n_models != batch)) {
    ctx->last_error = "assemble_kinematics: batch must equal the number of models (or use one shared model)";
    return PD_INVALID_ARGUMENT;
  }
  PD_CUDA(cudaSetDevice(ctx->device));
  const int n = ctx->n_links;
  Arena a;
  const size_t iq = a.add_in(q, sizeof(double) * n * batch);
  const size_t orel = a.add_out(rel, sizeof(double) * 12 * n * batch);
  const size_t obase = a.add_out(base_transport, sizeof(double) * 36 * batch);
  const size_t otr = a.add_out(transport, sizeof(double) * 36 * (n - 1) * batch);
  const size_t osc = a.add_out(screw, sizeof(double) * 6 * n * batch);
  pd_status st = a.stage(ctx);
  if (st != PD_OK) return st;
  launch_kinematics(ctx->raw.as<double>(), n, ctx->n_models, batch, a.in<double>(iq), a.out<double>(orel),
                    a.out<double>(obase), a.out<double>(otr), a.out<double>(osc), ctx->stream);
  ctx->launches++;
  return a.finish(ctx);
}

pd_status pd_link_inertias(pd_ctx* ctx, double* inertia) {
  if (!ctx) return PD_INVALID_ARGUMENT;
  if (bad_args(ctx, !inertia, "link_inertias: null buffer")) return PD_INVALID_ARGUMENT;
  if (ctx->n_models <= 0) {
    ctx->last_error = "link_inertias: no models set (pd_set_models)";
    return PD_INVALID_ARGUMENT;
  }
  pd_status cs = check_models(ctx, ctx->n_models, "link_inertias");
  if (cs != PD_OK) return cs;
  PD_CUDA(cudaSetDevice(ctx->device));
  const int64_t count = ctx->n_models * ctx->n_links;
  Arena a;
  const size_t o = a.add_out(inertia, sizeof(double) * 36 * count);
  pd_status st = a.stage(ctx);
  if (st != PD_OK) return st;
  launch_link_inertias(ctx->raw.as<double>(), count, a.out<double>(o), ctx->stream);
  ctx->launches++;
  return a.finish(ctx);
}

pd_status pd_articulated_body_inertias(pd_ctx* ctx, int64_t batch, int32_t n, const double* transport,
                                       const double* inertia, int32_t shared_inertia, const double* screw,
                                       double* abi, double* joint_inertia, double* gain, int32_t* slot_status,
                                       int32_t* slot_index) {
  if (!ctx) return PD_INVALID_ARGUMENT;
  if (bad_args(ctx, batch < 0 || n < 1 || (batch > 0 && (!inertia || !screw || !abi || !joint_inertia || !gain ||
                                                          (n > 1 && !transport))),
               "articulated_body_inertias: need n >= 1 and non-null buffers"))
    return PD_INVALID_ARGUMENT;
  if (batch == 0) return PD_OK;
  PD_CUDA(cudaSetDevice(ctx->device));
  const int64_t ib = shared_inertia ? 1 : batch;
  Arena a;
  const size_t itr = a.add_in(transport, sizeof(double) * 36 * (n - 1) * batch);
  const size_t iin = a.add_in(inertia, sizeof(double) * 36 * n * ib);
  const size_t isc = a.add_in(screw, sizeof(double) * 6 * n * batch);
  const size_t oab = a.add_out(abi, sizeof(double) * 36 * n * batch);
  const size_t oji = a.add_out(joint_inertia, sizeof(double) * n * batch);
  const size_t oga = a.add_out(gain, sizeof(double) * 6 * n * batch);
  const size_t ost = a.add_out(slot_status, sizeof(int32_t) * batch);
  const size_t oix = a.add_out(slot_index, sizeof(int32_t) * batch);
  pd_status st = a.stage(ctx);
  if (st != PD_OK) return st;
  launch_abi(batch, n, a.in<double>(itr), a.in<double>(iin), shared_inertia ? 0 : 36 * (int64_t)n, a.in<double>(isc),
             a.out<double>(oab), a.out<double>(oji), a.out<double>(oga), a.out<int32_t>(ost), a.out<int32_t>(oix),
             ctx->stream);
  ctx->launches++;
  return a.finish(ctx);
}

pd_status pd_constraint_basis(pd_ctx* ctx, int64_t count, const double* screw, double* basis) {
  if (!ctx) return PD_INVALID_ARGUMENT;
  if (bad_args(ctx, count < 0 || (count > 0 && (!screw || !basis)), "build_constraint_basis: null buffer"))
    return PD_INVALID_ARGUMENT;
  if (count == 0) return PD_OK;
  PD_CUDA(cudaSetDevice(ctx->device));
  Arena a;
  const size_t isc = a.add_in(screw, sizeof(double) * 6 * count);
  const size_t ob = a.add_out(basis, sizeof(double) * 30 * count);
  pd_status st = a.stage(ctx);
  if (st != PD_OK) return st;
  launch_basis(count, a.in<double>(isc), a.out<double>(ob), ctx->stream);
  ctx->launches++;
  return a.finish(ctx);
}

pd_status pd_cfa_operators(pd_ctx* ctx, int64_t batch, int32_t n, const double* inertia, int32_t shared_inertia,
                           const double* transport, const double* screw, const double* basis, double* constraint_diag,
                           double* constraint_upper, double* cross_sub, double* cross_diag, double* cross_super,
                           double* joint_diag, double* joint_off, int32_t* slot_status, int32_t* slot_index) {
  if (!ctx) return PD_INVALID_ARGUMENT;
  if (bad_args(ctx, batch < 0 || n < 1 || (batch > 0 && (!inertia || !screw || !basis || !constraint_diag ||
                                                          !cross_diag || !joint_diag ||
                                                          (n > 1 && (!transport || !constraint_upper || !cross_sub ||
                                                                     !cross_super || !joint_off)))),
               "build_cfa_operators: need n >= 1 and non-null buffers"))
    return PD_INVALID_ARGUMENT;
  if (batch == 0) return PD_OK;
  PD_CUDA(cudaSetDevice(ctx->device));
  const int64_t ib = shared_inertia ? 1 : batch, e = (int64_t)(n - 1) * batch, r = (int64_t)n * batch;
  Arena a;
  const size_t iin = a.add_in(inertia, sizeof(double) * 36 * n * ib);
  const size_t itr = a.add_in(transport, sizeof(double) * 36 * e);
  const size_t isc = a.add_in(screw, sizeof(double) * 6 * r);
  const size_t iba = a.add_in(basis, sizeof(double) * 30 * r);
  const size_t od = a.add_out(constraint_diag, sizeof(double) * 25 * r);
  const size_t ou = a.add_out(constraint_upper, sizeof(double) * 25 * e);
  const size_t obs = a.add_out(cross_sub, sizeof(double) * 5 * e);
  const size_t obd = a.add_out(cross_diag, sizeof(double) * 5 * r);
  const size_t obp = a.add_out(cross_super, sizeof(double) * 5 * e);
  const size_t ocd = a.add_out(joint_diag, sizeof(double) * r);
  const size_t oco = a.add_out(joint_off, sizeof(double) * e);
  const size_t obad = a.add_out(nullptr, sizeof(int32_t) * batch);
  pd_status st = a.stage(ctx);
  if (st != PD_OK) return st;
  int32_t* bad = a.out<int32_t>(obad);
  launch_cfa_ops(batch, n, a.in<double>(iin), shared_inertia ? 0 : 36 * (int64_t)n, a.in<double>(itr),
                 a.in<double>(isc), a.in<double>(iba), a.out<double>(od), a.out<double>(ou), a.out<double>(obs),
                 a.out<double>(obd), a.out<double>(obp), a.out<double>(ocd), a.out<double>(oco), bad, ctx->stream);
  ctx->launches += 2;
  st = a.finish(ctx);
  if (st != PD_OK) return st;
  std::vector<int32_t> hb(batch);
  PD_CUDA(cudaMemcpy(hb.data(), bad, sizeof(int32_t) * batch, cudaMemcpyDeviceToHost));
  for (int64_t p = 0; p < batch; ++p) {  // a link LLT failure: forward_dynamics.cpp:317-320
    if (slot_status) slot_status[p] = hb[p] < n ? PD_SLOT_LINK_INERTIA_NOT_PD : PD_SLOT_OK;
    if (slot_index) slot_index[p] = hb[p] < n ? hb[p] : 0;
  }
  return PD_OK;
}

pd_status pd_cfa_apply(pd_ctx* ctx, int32_t op, int64_t batch, int32_t n, const double* cross_sub,
                       const double* cross_diag, const double* cross_super, const double* joint_diag,
                       const double* joint_off, const double* in, double* out) {
  if (!ctx) return PD_INVALID_ARGUMENT;
  const bool joint = op == PD_APPLY_JOINT;
  if (bad_args(ctx, op < PD_APPLY_CROSS || op > PD_APPLY_JOINT || batch < 0 || n < 1 ||
                        (batch > 0 && (!in || !out || (joint ? !joint_diag || (n > 1 && !joint_off)
                                                              : !cross_diag || (n > 1 && (!cross_sub || !cross_super))))),
               "CfaOperators apply: invalid arguments"))
    return PD_INVALID_ARGUMENT;
  if (batch == 0) return PD_OK;
  PD_CUDA(cudaSetDevice(ctx->device));
  const int64_t e = (int64_t)(n - 1) * batch, r = (int64_t)n * batch;
  Arena a;
  const size_t ibs = a.add_in(joint ? nullptr : cross_sub, joint ? 0 : sizeof(double) * 5 * e);
  const size_t ibd = a.add_in(joint ? nullptr : cross_diag, joint ? 0 : sizeof(double) * 5 * r);
  const size_t ibp = a.add_in(joint ? nullptr : cross_super, joint ? 0 : sizeof(double) * 5 * e);
  const size_t icd = a.add_in(joint ? joint_diag : nullptr, joint ? sizeof(double) * r : 0);
  const size_t ico = a.add_in(joint ? joint_off : nullptr, joint ? sizeof(double) * e : 0);
  const size_t iv = a.add_in(in, sizeof(double) * r * (op == PD_APPLY_CROSS_TRANSPOSE ? 5 : 1));
  const size_t ov = a.add_out(out, sizeof(double) * r * (op == PD_APPLY_CROSS ? 5 : 1));
  pd_status st = a.stage(ctx);
  if (st != PD_OK) return st;
  launch_cfa_apply(op, batch, n, a.in<double>(ibs), a.in<double>(ibd), a.in<double>(ibp), a.in<double>(icd),
                   a.in<double>(ico), a.in<double>(iv), a.out<double>(ov), ctx->stream);
  ctx->launches++;
  return a.finish(ctx);
}

}  // extern "C"

extern "C" {

pd_status pd_host_alloc(uint64_t bytes, void** out) {
  if (!out) return PD_INVALID_ARGUMENT;
  *out = nullptr;
  if (bytes == 0) return PD_OK;
  return cudaMallocHost(out, (size_t)bytes) == cudaSuccess ? PD_OK : PD_CUDA_ERROR;
}

void pd_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

}  // extern "C"

extern "C" {

pd_status pd_propagate(pd_ctx* ctx, int32_t kind, int64_t batch, int32_t n, const double* base_transport,
                       const double* transport, const double* screw, const double* inertia, int32_t shared_inertia,
                       const double* qdot, const double* qddot, const double* velocity, const double* acceleration,
                       const double* boundary, double* out) {
  if (!ctx) return PD_INVALID_ARGUMENT;
  const bool vel = kind == PD_PROPAGATE_VELOCITIES, acc = kind == PD_PROPAGATE_ACCELERATIONS,
             frc = kind == PD_PROPAGATE_FORCES;
  if (bad_args(ctx, (!vel && !acc && !frc) || batch < 0 || n < 1 ||
                        (batch > 0 && (!screw || !out || !boundary || (n > 1 && !transport) ||
                                       ((vel || acc) && (!base_transport || !qdot)) || (acc && (!qddot || !velocity)) ||
                                       (frc && (!inertia || !velocity || !acceleration)))),
               "propagate: invalid arguments"))
    return PD_INVALID_ARGUMENT;
  if (batch == 0) return PD_OK;
  PD_CUDA(cudaSetDevice(ctx->device));
  const int64_t e = (int64_t)(n - 1) * batch, r = (int64_t)n * batch;
  Arena a;
  const size_t ib = a.add_in(vel || acc ? base_transport : nullptr, vel || acc ? sizeof(double) * 36 * batch : 0);
  const size_t it = a.add_in(transport, sizeof(double) * 36 * e);
  const size_t is = a.add_in(screw, sizeof(double) * 6 * r);
  const size_t ij = a.add_in(frc ? inertia : nullptr, frc ? sizeof(double) * 36 * n * (shared_inertia ? 1 : batch) : 0);
  const size_t iq = a.add_in(vel || acc ? qdot : nullptr, vel || acc ? sizeof(double) * r : 0);
  const size_t iqq = a.add_in(acc ? qddot : nullptr, acc ? sizeof(double) * r : 0);
  const size_t iv = a.add_in(acc || frc ? velocity : nullptr, acc || frc ? sizeof(double) * 6 * r : 0);
  const size_t ia = a.add_in(frc ? acceleration : nullptr, frc ? sizeof(double) * 6 * r : 0);
  const size_t ibd = a.add_in(boundary, sizeof(double) * 6);
  const size_t oc = a.add_out(nullptr, sizeof(double) * 36 * e);
  const size_t orh = a.add_out(nullptr, sizeof(double) * 6 * r);
  const size_t ox = a.add_out(out, sizeof(double) * 6 * r);
  pd_status st = a.stage(ctx);
  if (st != PD_OK) return st;
  launch_propagate_setup(kind, batch, n, a.in<double>(ib), a.in<double>(it), a.in<double>(is), a.in<double>(ij),
                         shared_inertia ? 0 : 36 * (int64_t)n, a.in<double>(iq), a.in<double>(iqq), a.in<double>(iv),
                         a.in<double>(ia), a.in<double>(ibd), a.out<double>(oc), a.out<double>(orh), ctx->stream);
  launch_bidiag6(a.out<double>(oc), a.out<double>(orh), a.out<double>(ox), batch, n, frc ? 1 : 0, ctx->stream);
  ctx->launches += 2;
  return a.finish(ctx);
}

}  // extern "C"
