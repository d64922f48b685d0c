// capi.cu -- the C ABI of include/boysfn_b200.h: table handles, kernel
// dispatch, the host paths behind boys_batch_many (a one-kernel path over
// host-mapped buffers for small batches, a chunked three-stream pipeline for
// large ones, optionally sharded over several devices), and the
// synthetic-workload generators.  Every evaluation runs on the GPU; there is no
// CPU fallback: without a device the calls return BOYSFN_ERR_CUDA.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only; ranges cost nothing without a profiler attached

#include <emmintrin.h>  // SSE2 non-temporal stores (host copy out of pinned staging)

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/boysfn_b200.h"
#include "boys_launch.h"
#include "capi_internal.h"
#include "embedded_tables.inc"

using boysfn_dev::EvalParams;
using boysfn_dev::kMaxCoef;

// ----------------------------------------------------------------- errors --
namespace {

// Exact reference wording (eval.cpp:14-17,51,90-91; tables.cpp:15-28).
constexpr const char* kMsgSize = "boys_batch_many: output span has wrong size";
constexpr const char* kMsgDomain = "boys_batch: x must be finite and non-negative";
constexpr const char* kMsgRange = "boys_batch: k out of range for this table set";
constexpr const char* kMsgUpward = "upward_recursion: x must be positive";

thread_local std::string t_last_error;
std::atomic<unsigned long long> g_launches{0};

}  // namespace

int boysfn_internal::fail(int status, const std::string& msg) {
  t_last_error = msg;
  return status;
}

int boysfn_internal::cuda_fail(cudaError_t e, const char* where) {
  t_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return BOYSFN_ERR_CUDA;
}

void boysfn_internal::count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

using boysfn_internal::cuda_fail;
using boysfn_internal::fail;

namespace {

bool fill_rational(const boysfn_rational_desc& r, double* num, double* den) {
  if (r.n > kMaxCoef - 1 || r.m > kMaxCoef - 1) return false;
  std::fill(num, num + kMaxCoef, 0.0);
  std::fill(den, den + kMaxCoef, 0.0);
  std::copy(r.numer, r.numer + r.n + 1, num);
  std::copy(r.denom, r.denom + r.m + 1, den);
  return true;
}

// validate_tables (tables.cpp:14-32), same order and messages.
int validate_desc(const boysfn_table_desc* d) {
  if (d->k_max < 0) return fail(BOYSFN_ERR_TABLES, "tables: k_max must be non-negative");
  if (!(d->eps_tol > 0)) return fail(BOYSFN_ERR_TABLES, "tables: eps_tol must be positive");
  if (!(d->x0 > 0 && d->x0 < d->x1)) return fail(BOYSFN_ERR_TABLES, "tables: need 0 < x0 < x1");
  if (d->r_A == nullptr)
    return fail(BOYSFN_ERR_TABLES, "tables: need exactly k_max+1 region-A tables");
  auto check = [](const boysfn_rational_desc& r, const std::string& what) -> int {
    if (r.n < 0 || r.m < 0 || r.numer == nullptr || r.denom == nullptr)
      return fail(BOYSFN_ERR_TABLES, "tables: empty coefficient vector in " + what);
    for (int i = 0; i <= r.n; ++i)
      if (!std::isfinite(r.numer[i])) return fail(BOYSFN_ERR_TABLES, "tables: non-finite value in " + what);
    for (int i = 0; i <= r.m; ++i)
      if (!std::isfinite(r.denom[i])) return fail(BOYSFN_ERR_TABLES, "tables: non-finite value in " + what);
    if (r.denom[r.m] != 1.0)
      return fail(BOYSFN_ERR_TABLES, "tables: non-monic denominator in " + what);
    return BOYSFN_OK;
  };
  if (int st = check(d->r_B, "r_B")) return st;
  for (int k = 0; k <= d->k_max; ++k)
    if (int st = check(d->r_A[k], "r_A[" + std::to_string(k) + "]")) return st;
  return BOYSFN_OK;
}

// What the device image needs to evaluate a set (eval.cpp itself never
// validates): k_max >= 0, k_max + 1 region-A tables, non-empty finite
// coefficient vectors.  Messages as validate_tables' for the same faults.
// Degrees above 23 are accepted here and refused per order at launch.
int check_device_desc(const boysfn_table_desc* d) {
  if (d->k_max < 0) return fail(BOYSFN_ERR_TABLES, "tables: k_max must be non-negative");
  if (d->r_A == nullptr)
    return fail(BOYSFN_ERR_TABLES, "tables: need exactly k_max+1 region-A tables");
  auto check = [](const boysfn_rational_desc& r, const std::string& what) -> int {
    if (r.n < 0 || r.m < 0 || r.numer == nullptr || r.denom == nullptr)
      return fail(BOYSFN_ERR_TABLES, "tables: empty coefficient vector in " + what);
    for (int i = 0; i <= r.n; ++i)
      if (!std::isfinite(r.numer[i])) return fail(BOYSFN_ERR_TABLES, "tables: non-finite value in " + what);
    for (int i = 0; i <= r.m; ++i)
      if (!std::isfinite(r.denom[i])) return fail(BOYSFN_ERR_TABLES, "tables: non-finite value in " + what);
    return BOYSFN_OK;
  };
  if (int st = check(d->r_B, "r_B")) return st;
  for (int k = 0; k <= d->k_max; ++k)
    if (int st = check(d->r_A[k], "r_A[" + std::to_string(k) + "]")) return st;
  return BOYSFN_OK;
}

int build_handle(const boysfn_table_desc* d, boysfn_tables_s* h) {
  h->x0 = d->x0;
  h->x1 = d->x1;
  h->eps_tol = d->eps_tol;
  h->k_max = d->k_max;
  const int kdev = d->k_max;
  h->params.assign(kdev + 1, EvalParams{});
  h->variant.assign(kdev + 1, boysfn_dev::kVariantPadded);
  h->degree_ok.assign(kdev + 1, 0);
  h->deg_na.assign(kdev + 1, 0);
  h->deg_ma.assign(kdev + 1, 0);
  h->deg_nb = d->r_B.n;
  h->deg_mb = d->r_B.m;
  for (int k = 0; k <= kdev; ++k) {
    h->deg_na[k] = d->r_A[k].n;
    h->deg_ma[k] = d->r_A[k].m;
    EvalParams& p = h->params[k];
    p.x0 = d->x0;
    p.x1 = d->x1;
    const bool ok = fill_rational(d->r_A[k], p.numA, p.denA) && fill_rational(d->r_B, p.numB, p.denB);
    h->degree_ok[k] = ok ? 1 : 0;
    int na, ma, nb, mb;
    boysfn_dev::embedded_degrees(k, &na, &ma, &nb, &mb);
    if (d->r_A[k].n == na && d->r_A[k].m == ma && d->r_B.n == nb && d->r_B.m == mb)
      h->variant[k] = boysfn_dev::kVariantEmbedded;
    else if (d->r_A[k].n <= boysfn_dev::kCompactNA && d->r_A[k].m <= boysfn_dev::kCompactMA &&
             d->r_B.n <= boysfn_dev::kCompactNB && d->r_B.m <= boysfn_dev::kCompactMB)
      h->variant[k] = boysfn_dev::kVariantCompact;
  }
  return BOYSFN_OK;
}

boysfn_tables_s* embedded_handle() {
  static boysfn_tables_s* h = [] {
    std::vector<boysfn_rational_desc> ra(BOYSFN_EMB_KMAX + 1);
    for (int k = 0; k <= BOYSFN_EMB_KMAX; ++k)
      ra[k] = boysfn_rational_desc{kEmbDegA[k][0], kEmbDegA[k][1], kEmbNumA[k], kEmbDenA[k]};
    boysfn_table_desc d{BOYSFN_EMB_X0, BOYSFN_EMB_X1, BOYSFN_EMB_KMAX, BOYSFN_EMB_EPS,
                        boysfn_rational_desc{kEmbDegB[0], kEmbDegB[1], kEmbNumB, kEmbDenB},
                        ra.data()};
    auto* t = new boysfn_tables_s;
    build_handle(&d, t);
    t->is_embedded = true;
    return t;
  }();
  return h;
}

// ------------------------------------------------------------- dispatch --
struct DeviceInfo {
  int sms = 0;
  std::map<std::pair<const void*, size_t>, int> blocks_per_sm;  // (kernel, dynamic smem)
  cudaMemPool_t pool = nullptr;  // this library's stream-ordered pool
};

std::mutex g_dev_mu;
std::map<int, DeviceInfo> g_devices;

// The library's own stream-ordered memory pool on the current device (for the
// per-launch scheduler counters and Algorithm 2's scratch).  Unlike the
// device's default pool it keeps up to 64 MB reserved across synchronisations,
// so a launch after a sync does not re-map physical memory, and setting that
// does not change the default pool the rest of the process uses.
int device_pool(cudaMemPool_t* out) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_dev_mu);
  DeviceInfo& di = g_devices[dev];
  if (di.pool == nullptr) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    CUDA_TRY(cudaMemPoolCreate(&di.pool, &props));
    uint64_t keep = uint64_t(64) << 20;
    CUDA_TRY(cudaMemPoolSetAttribute(di.pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  *out = di.pool;
  return BOYSFN_OK;
}

// Zeroed per-launch counter in stream order: the caller's (a pipeline slot's
// own, reused on its private stream) or one from the library pool, released
// after the launch in stream order (*release set).
int launch_counter(unsigned long long* given, cudaStream_t stream, unsigned long long** ctr, bool* release) {
  *release = given == nullptr;
  if (given != nullptr) {
    *ctr = given;
  } else {
    cudaMemPool_t pool = nullptr;
    if (int st = device_pool(&pool)) return st;
    CUDA_TRY(cudaMallocFromPoolAsync(reinterpret_cast<void**>(ctr), sizeof(unsigned long long), pool, stream));
  }
  CUDA_TRY(cudaMemsetAsync(*ctr, 0, sizeof(unsigned long long), stream));
  return BOYSFN_OK;
}

int occupancy(const void* fn, int threads, size_t smem, int* sms, int* bps) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_dev_mu);
  DeviceInfo& di = g_devices[dev];
  if (di.sms == 0) CUDA_TRY(cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev));
  auto it = di.blocks_per_sm.find({fn, smem});
  if (it == di.blocks_per_sm.end()) {
    // the whole unified L1/shared array as shared memory: these kernels stream
    // (no L1 reuse) and their resident blocks are often shared-memory bound
    if (std::getenv("BOYSFN_DEFAULT_CARVEOUT") == nullptr)
      CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    cudaSharedmemCarveoutMaxShared));
    if (smem > 48 * 1024) {  // opt in to the larger of this and any earlier request
      cudaFuncAttributes fa;
      CUDA_TRY(cudaFuncGetAttributes(&fa, fn));
      if (static_cast<size_t>(fa.maxDynamicSharedSizeBytes) < smem)
        CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    }
    int b = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, threads, smem));
    it = di.blocks_per_sm.emplace(std::make_pair(fn, smem), std::max(b, 1)).first;
  }
  *sms = di.sms;
  *bps = it->second;
  return BOYSFN_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 2D map over the SoA output: dim0 = x index (n, contiguous), dim1 = order
// (k+1 rows, stride ld); box = one block tile, 128 x by k+1 rows.
bool make_soa_tmap(CUtensorMap* m, double* out, size_t n, size_t ld, int R, int box_x) {
  EncodeTiledFn enc = encode_tiled();
  if (enc == nullptr || (reinterpret_cast<uintptr_t>(out) & 15) || (ld * sizeof(double)) % 16 ||
      n > (size_t(1) << 31) - 256)
    return false;
  const cuuint64_t dims[2] = {n, static_cast<cuuint64_t>(R)};
  const cuuint64_t strides[1] = {ld * sizeof(double)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_x), static_cast<cuuint32_t>(R)};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, out, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tensor-map coordinates are int32: tensor-store launches above this many x
// are split (launch_eval).
constexpr size_t kTmaMaxX = (size_t(1) << 31) - (size_t(1) << 20);

// 2D map over the AoS output for the run-time-k kernel's padded stage: dim0 =
// order (R, contiguous), dim1 = row (stride 8R B); box = pitch x rows, so the
// stage's pad columns (>= R) are outside the map and clipped by the store.
bool make_aos_pad_tmap(CUtensorMap* m, double* out, size_t n, int R, int pitch, int rows) {
  EncodeTiledFn enc = encode_tiled();
  if (enc == nullptr || (reinterpret_cast<uintptr_t>(out) & 15) || (R * sizeof(double)) % 16 ||
      (pitch * sizeof(double)) % 16 || pitch > 256 || n > (size_t(1) << 31) - 256)
    return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(R), n};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(R) * sizeof(double)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(pitch), static_cast<cuuint32_t>(rows)};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, out, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Output-path selection (interleaved medians of
// the candidate paths at every k on one B200, profiles/r01_path_sweep.txt and
// profiles/r02_path_policy.txt).  Large k is HBM-write-bound and wants long
// contiguous write bursts: block tiles of 256 x stored by the TMA engine (2 KB
// SoA row segments / 2 KB*(k+1) AoS spans).  Around k = 6..9 the FP64 work per
// byte is highest and the A/B/C divergence costs most: the 128-x tiles sorted
// by region first.  Small k is issue-bound and wants no divergence at the
// least overhead: the per-warp region-binned kernels.  AoS stages whose rows
// are a multiple of 4 doubles are padded by 2 (conflict-free STS.128) and
// stored through a 2D tensor map that clips the pad (aos_stage_pitch).
//   SoA: k <= 5 binned; 6..9 block-TMA region-sorted; else block-TMA
//        (rows off a 32-B sector boundary: the shifted per-row bulk store)
//   AoS: k <= 5 binned; 6..8 block-TMA region-sorted; else block-TMA
//        (transpose if the output is not 16-B aligned or no tensor map applies)
int choose_store(int layout, int k, const double* d_out) {
  const int R = k + 1;
  const char* e = std::getenv(layout == BOYSFN_LAYOUT_SOA ? "BOYSFN_SOA_PATH" : "BOYSFN_AOS_PATH");
  const std::string want = e ? e : "";
  const bool a16 = (reinterpret_cast<uintptr_t>(d_out) & 15) == 0;
  if (layout == BOYSFN_LAYOUT_SOA) {
    if (want == "warp") return boysfn_dev::kStoreSoA;
    if (want == "block") return boysfn_dev::kStoreSoABlock;
    if (want == "binned") return boysfn_dev::kStoreSoABinned;
    if (want == "blocktma") return boysfn_dev::kStoreSoABlockTma;
    if (want == "blocktmabin") return boysfn_dev::kStoreSoABlockTmaBin;
    if (want == "blockbulk") return boysfn_dev::kStoreSoABlockBulk;
    if (want == "blockbulkw") return k <= boysfn_dev::kSoAWideKmax ? boysfn_dev::kStoreSoABlockBulkW : boysfn_dev::kStoreSoABlockBulk;
    if (want == "blockbulkw3") return boysfn_dev::kStoreSoABlockBulkW3;
    if (k <= 5) return boysfn_dev::kStoreSoABinned;
    return k <= 9 ? boysfn_dev::kStoreSoABlockTmaBin : boysfn_dev::kStoreSoABlockTma;
  }
  if (want == "xpose") return boysfn_dev::kStoreAoSXpose;
  if (want == "binned") return boysfn_dev::kStoreAoSBinned;
  if (want == "blocktma" && a16) return boysfn_dev::kStoreAoSBlockTma;
  if (want == "blocktmabin" && a16) return boysfn_dev::kStoreAoSBlockTmaBin;
  if (!want.empty()) return boysfn_dev::kStoreAoSXpose;
  if (k <= 5) return boysfn_dev::kStoreAoSBinned;
  if (!a16) return boysfn_dev::kStoreAoSXpose;
  return k <= 8 ? boysfn_dev::kStoreAoSBlockTmaBin : boysfn_dev::kStoreAoSBlockTma;
}

// BOYSFN_GENERIC=1 routes every order through the run-time-k kernels (by the
// policy below), =2 through the per-warp one, =3 the staged block kernel, =4
// the register-buffered block kernel (tests and experiments).
int generic_forced() {
  const char* e = std::getenv("BOYSFN_GENERIC");
  return e != nullptr && e[0] >= '1' && e[0] <= '4' ? e[0] - '0' : 0;
}
// Up to this order the staged block kernel (F written into the stage as it is
// produced, 40 registers) beats the register-buffered one (F in registers
// while the previous tile drains, 124-165 registers); profiles/r01_generic_kernel.txt.
constexpr int kGenericStageKmax = 34;

// The run-time-k kernels: orders above 32 and forced regions above 32.  Block
// tiles stored by the TMA engine where a tensor map / bulk copy applies,
// otherwise (unaligned or strided output, a forced region, host-mapped
// output) the per-warp kernel.
int launch_generic(const boysfn_tables_s* t, const double* d_x, size_t n, int k, double* d_out, int layout,
                   size_t ld, cudaStream_t stream, unsigned long long* d_bad, int force_region,
                   unsigned long long* d_ctr = nullptr, bool allow_tma = true) {
  const int R = k + 1;
  EvalParams p = t->params[k];
  int na = t->deg_na[k], ma = t->deg_ma[k], nb = t->deg_nb, mb = t->deg_mb;
  const int mode = generic_forced();
  if (allow_tma && force_region < 0 && mode != 2) {
    const bool soa = layout == BOYSFN_LAYOUT_SOA;
    CUtensorMap tmap;
    std::memset(&tmap, 0, sizeof tmap);
    const bool ok = soa ? make_soa_tmap(&tmap, d_out, n, ld, R, boysfn_dev::kGenericTileX)
                        : (reinterpret_cast<uintptr_t>(d_out) & 15) == 0;
    const bool staged = mode == 3 || (mode != 4 && k <= kGenericStageKmax);
    const void* fn = staged ? boysfn_dev::kernel_generic_stage(soa) : boysfn_dev::kernel_generic_tma(k, soa);
    if (ok && fn != nullptr) {
      const int pitch = staged ? R : boysfn_dev::generic_stage_pitch(soa, R);
      int pad_tmap = 0;
      if (!soa && pitch != R && std::getenv("BOYSFN_GENERIC_AOS_ROWS") == nullptr)
        pad_tmap = make_aos_pad_tmap(&tmap, d_out, n, R, pitch, boysfn_dev::kGenericTileX) ? 1 : 0;
      const size_t smem =
          boysfn_dev::block_tma_smem_bytes<boysfn_dev::kStoreSoABlockTmaBin>(pitch, boysfn_dev::kGenericTileX);
      int sms = 0, bps = 0;
      if (int st = occupancy(fn, boysfn_dev::kGenericTileX, smem, &sms, &bps)) return st;
      const size_t ntiles = (n + boysfn_dev::kGenericTileX - 1) / boysfn_dev::kGenericTileX;
      const unsigned grid = static_cast<unsigned>(std::min<size_t>(ntiles, static_cast<size_t>(sms) * bps));
      unsigned long long* counter = nullptr;
      bool release = false;
      if (int st = launch_counter(d_ctr, stream, &counter, &release)) return st;
      void* args[] = {&p, &na, &ma, &nb, &mb, &k, &d_x, &n, &d_out, &d_bad, &counter, &tmap, &pad_tmap, &ld};
      const cudaError_t le = cudaLaunchKernel(fn, dim3(grid), dim3(boysfn_dev::kGenericTileX), args, smem, stream);
      if (release) CUDA_TRY(cudaFreeAsync(counter, stream));
      if (le != cudaSuccess) return cuda_fail(le, "cudaLaunchKernel");
      boysfn_internal::count_launch();
      return BOYSFN_OK;
    }
  }
  const void* fn = boysfn_dev::kernel_generic();
  const int aos_flag = layout == BOYSFN_LAYOUT_AOS ? 1 : 0;
  const size_t smem = aos_flag ? sizeof(double) * boysfn_dev::kThreadsPerBlock *
                                     boysfn_dev::generic_aos_pitch(k + 1)
                               : 0;  // per-warp AoS stage, 32 rows x odd pitch
  int sms = 0, bps = 0;
  if (int st = occupancy(fn, boysfn_dev::kThreadsPerBlock, smem, &sms, &bps)) return st;
  const size_t want = ((n + 31) / 32 + boysfn_dev::kWarpsPerBlock - 1) / boysfn_dev::kWarpsPerBlock;
  const unsigned grid = static_cast<unsigned>(std::min<size_t>(want, static_cast<size_t>(sms) * bps));
  int aos = aos_flag;
  unsigned long long* counter = nullptr;
  bool release = false;
  if (int st = launch_counter(d_ctr, stream, &counter, &release)) return st;
  void* args[] = {&p, &na, &ma, &nb, &mb, &k, &force_region, &d_x, &n, &d_out, &ld, &aos, &d_bad, &counter};
  const cudaError_t le = cudaLaunchKernel(fn, dim3(grid), dim3(boysfn_dev::kThreadsPerBlock), args, smem, stream);
  if (release) CUDA_TRY(cudaFreeAsync(counter, stream));
  if (le != cudaSuccess) return cuda_fail(le, "cudaLaunchKernel");
  boysfn_internal::count_launch();
  return BOYSFN_OK;
}

bool tensor_store(int store, int R) {
  return store == boysfn_dev::kStoreSoABlockTma || store == boysfn_dev::kStoreSoABlockTmaBin ||
         ((store == boysfn_dev::kStoreAoSBlockTma || store == boysfn_dev::kStoreAoSBlockTmaBin) &&
          boysfn_dev::aos_stage_pitch(R) != R);
}

int launch_store(const boysfn_tables_s* t, const double* d_x, size_t n, int k, double* d_out, int layout,
                 size_t ld, cudaStream_t stream, unsigned long long* d_bad, unsigned long long* d_ctr, int store,
                 unsigned long long ibase);

// Launches the evaluation kernel; k already validated against the handle.
// force_store >= 0 overrides the path choice (the host API's small-batch path
// writes host-mapped memory and takes the per-warp LSU stores).  Tensor-map
// stores address x by int32 coordinates: batches above kTmaMaxX are split
// into consecutive launches on the stream (the first-bad index stays global).
int launch_eval(const boysfn_tables_s* t, const double* d_x, size_t n, int k, double* d_out,
                int layout, size_t ld, cudaStream_t stream, unsigned long long* d_bad,
                unsigned long long* d_ctr = nullptr, int force_store = -1) {
  if (n == 0) return BOYSFN_OK;
  if (!t->degree_ok[k])
    return fail(BOYSFN_ERR_UNSUPPORTED, "table degree exceeds the device image (max 23)");
  if (k > BOYSFN_DEVICE_KMAX_RT)
    return fail(BOYSFN_ERR_UNSUPPORTED, "order above the run-time-k kernels' bound (64)");
  if (k > boysfn_dev::kKernelKmax || generic_forced())
    return launch_generic(t, d_x, n, k, d_out, layout, ld, stream, d_bad, -1, d_ctr, force_store < 0);
  // k = 0: the AoS and SoA outputs are the same n doubles; take the SoA
  // kernels (0.327 against 0.341 ms at 1e8 x) unless a path is forced
  if (k == 0 && layout == BOYSFN_LAYOUT_AOS && force_store < 0 && std::getenv("BOYSFN_AOS_PATH") == nullptr) {
    layout = BOYSFN_LAYOUT_SOA;
    ld = n;
  }
  const int store = force_store >= 0 ? force_store : choose_store(layout, k, d_out);
  if (!tensor_store(store, k + 1) || n <= kTmaMaxX)
    return launch_store(t, d_x, n, k, d_out, layout, ld, stream, d_bad, d_ctr, store, 0);
  const size_t R = static_cast<size_t>(k) + 1;
  for (size_t off = 0; off < n; off += kTmaMaxX) {
    const size_t m = std::min(kTmaMaxX, n - off);
    double* o = layout == BOYSFN_LAYOUT_SOA ? d_out + off : d_out + off * R;
    if (int st = launch_store(t, d_x + off, m, k, o, layout, ld, stream, d_bad, d_ctr, store, off)) return st;
  }
  return BOYSFN_OK;
}

int launch_store(const boysfn_tables_s* t, const double* d_x, size_t n, int k, double* d_out, int layout,
                 size_t ld, cudaStream_t stream, unsigned long long* d_bad, unsigned long long* d_ctr, int store,
                 unsigned long long ibase) {
  const int R = k + 1;
  const int v = t->variant[k];
  const void* fn = nullptr;
  size_t smem = 0;
  CUtensorMap tmap;
  std::memset(&tmap, 0, sizeof tmap);
  // the tensor store for rows that start on a 32-B sector boundary (output
  // 32-B aligned, ld a multiple of 4); otherwise the same tile kernel with
  // per-row bulk copies whose windows are shifted to the row's sector phase
  // (any ld, any 8-B alignment): at ld = 2 mod 4 it beats the tensor store
  // (k = 32: 0.89 vs 0.86, k = 8: 0.96 vs 0.91 of the ld = n rate,
  // profiles/r02_tma_edges.txt)
  // (BOYSFN_SOA_PATH=blocktma* forces the tensor store wherever its map encodes)
  const bool sector_rows = (reinterpret_cast<uintptr_t>(d_out) & 31) == 0 && (ld & 3) == 0;
  if (store == boysfn_dev::kStoreSoABlockTma || store == boysfn_dev::kStoreSoABlockTmaBin) {
    const bool want_tensor = sector_rows || std::getenv("BOYSFN_SOA_PATH") != nullptr;
    // (the 256-x plain tiles: 4-5% faster than the region-sorted 128-x ones
    // at k = 8..16 for these strides, profiles/r02_bulk_vs_bulkbin.txt)
    if (!want_tensor || !make_soa_tmap(&tmap, d_out, n, ld, R, boysfn_dev::block_tma_tile_x(store)))
      store = boysfn_dev::kStoreSoABlockBulk;
  }
  // rows off a 1-KB boundary at k = 10..24: the same bulk store with 512-x
  // tiles (boys_launch.h kSoAWideTileX)
  const bool kb_rows = (reinterpret_cast<uintptr_t>(d_out) & 1023) == 0 && (ld & 127) == 0;
  if ((store == boysfn_dev::kStoreSoABlockTma || store == boysfn_dev::kStoreSoABlockBulk) && !kb_rows &&
      k >= boysfn_dev::kSoAWideKmin && k <= boysfn_dev::kSoAWideKmax && std::getenv("BOYSFN_SOA_PATH") == nullptr)
    store = boysfn_dev::kStoreSoABlockBulkW;
  if (store == boysfn_dev::kStoreSoABlockBulk && k > boysfn_dev::kSoAWideKmax && std::getenv("BOYSFN_SOA_PATH") == nullptr)
    store = boysfn_dev::kStoreSoABlockBulkW3;
  if ((store == boysfn_dev::kStoreSoABlockBulk || store == boysfn_dev::kStoreSoABlockBulkW ||
       store == boysfn_dev::kStoreSoABlockBulkW3) &&
      (reinterpret_cast<uintptr_t>(d_out) & 7))
    store = boysfn_dev::kStoreSoABlock;
  if ((store == boysfn_dev::kStoreAoSBlockTma || store == boysfn_dev::kStoreAoSBlockTmaBin) &&
      boysfn_dev::aos_stage_pitch(R) != R &&
      !make_aos_pad_tmap(&tmap, d_out, n, R, boysfn_dev::aos_stage_pitch(R), boysfn_dev::block_tma_tile_x(store)))
    store = boysfn_dev::kStoreAoSXpose;
  const int threads = boysfn_dev::block_tma_tile_x(store);  // kThreadsPerBlock for the other kinds
  switch (store) {
    case boysfn_dev::kStoreSoABlockTma:
      fn = boysfn_dev::kernel_soa_block_tma(k, v);
      smem = boysfn_dev::block_tma_smem_bytes<boysfn_dev::kStoreSoABlockTma>(R, threads);
      break;
    case boysfn_dev::kStoreSoABlockBulk:
      fn = boysfn_dev::kernel_soa_block_bulk(k, v);
      smem = boysfn_dev::block_tma_smem_bytes<boysfn_dev::kStoreSoABlockBulk>(R, threads);
      break;
    case boysfn_dev::kStoreSoABlockBulkW:
      fn = boysfn_dev::kernel_soa_block_bulk_w(k, v);
      smem = boysfn_dev::block_tma_smem_bytes<boysfn_dev::kStoreSoABlockBulkW>(R, threads);
      break;
    case boysfn_dev::kStoreSoABlockBulkW3:
      fn = boysfn_dev::kernel_soa_block_bulk_w3(k, v);
      smem = boysfn_dev::block_tma_smem_bytes<boysfn_dev::kStoreSoABlockBulkW3>(R, threads);
      break;
    case boysfn_dev::kStoreAoSBlockTma:
      fn = boysfn_dev::kernel_aos_block_tma(k, v);
      smem = boysfn_dev::block_tma_smem_bytes<boysfn_dev::kStoreAoSBlockTma>(R, threads);
      break;
    case boysfn_dev::kStoreSoABlockTmaBin:
      fn = boysfn_dev::kernel_soa_block_tma_bin(k, v);
      smem = boysfn_dev::block_tma_smem_bytes<boysfn_dev::kStoreSoABlockTmaBin>(R, threads);
      break;
    case boysfn_dev::kStoreAoSBlockTmaBin:
      fn = boysfn_dev::kernel_aos_block_tma_bin(k, v);
      smem = boysfn_dev::block_tma_smem_bytes<boysfn_dev::kStoreAoSBlockTmaBin>(R, threads);
      break;
    case boysfn_dev::kStoreSoA:
      fn = boysfn_dev::kernel_soa(k, v);
      break;
    case boysfn_dev::kStoreAoSXpose:
      fn = boysfn_dev::kernel_aos_xpose(k, v);
      smem = sizeof(double) * boysfn_dev::kWarpsPerBlock * boysfn_dev::kXposePitch * R;
      break;
    case boysfn_dev::kStoreSoABlock:
      fn = boysfn_dev::kernel_soa_block(k, v);
      smem = sizeof(double) * boysfn_dev::kBlockX * R;
      break;
    case boysfn_dev::kStoreSoABinned:
      fn = boysfn_dev::kernel_soa_binned(k, v);
      smem = sizeof(double) * boysfn_dev::kWarpsPerBlock * boysfn_dev::binned_smem_doubles_per_warp(k, true);
      break;
    default:
      fn = boysfn_dev::kernel_aos_binned(k, v);
      smem = sizeof(double) * boysfn_dev::kWarpsPerBlock * boysfn_dev::binned_smem_doubles_per_warp(k, false);
      break;
  }
  int sms = 0, bps = 0;
  if (int st = occupancy(fn, threads, smem, &sms, &bps)) return st;
  const size_t ntiles = (n + 31) / 32;
  const size_t wpb = static_cast<size_t>(threads / 32);
  const size_t want = (ntiles + wpb - 1) / wpb;
  const unsigned grid = static_cast<unsigned>(std::min<size_t>(want, static_cast<size_t>(sms) * bps));
  EvalParams p = t->params[k];
  // Per-launch tile counter, zeroed and used in stream order, so concurrent
  // launches on other streams never share it.
  unsigned long long* counter = nullptr;
  bool release = false;
  if (int st = launch_counter(d_ctr, stream, &counter, &release)) return st;
  // the block-TMA kernels take the last two; the others ignore the extra entries
  void* args[] = {&p, &d_x, &n, &d_out, &ld, &d_bad, &counter, &tmap, &ibase};
  const cudaError_t le = cudaLaunchKernel(fn, dim3(grid), dim3(threads), args, smem, stream);
  if (release) CUDA_TRY(cudaFreeAsync(counter, stream));
  if (le != cudaSuccess) return cuda_fail(le, "cudaLaunchKernel");
  boysfn_internal::count_launch();
  return BOYSFN_OK;
}

// --------------------------------------------------------- host pipeline --
// Staging for one host call on one device: three slots, each with its own
// stream; a chunk's H2D copy, kernel and D2H copy follow one another on its
// slot's stream, and the slots overlap, so the link stays busy.  Every buffer
// is allocated on first use by the path that needs it (a small call never
// touches the chunk buffers), and pipelines come from a bounded per-device
// pool shared by all host threads (PipelinePool below).
struct Pipeline {
  static constexpr int kSlots = 3;
  static constexpr size_t kChunkOutBytes = size_t(256) << 20;  // profiles/r01_e2e_chunk.txt
  int device = -1;
  cudaStream_t stream[kSlots] = {};
  cudaEvent_t copied[kSlots] = {};  // D2H of the slot's chunk
  double* d_x[kSlots] = {};
  double* d_out[kSlots] = {};
  unsigned long long* d_ctr = nullptr;  // kSlots scheduler counters (slot s: only on stream[s])
  size_t cap_x = 0;                     // x capacity per slot (allocated)
  size_t cap_out = 0;                   // output doubles per slot (the chunk size; allocated lazily)
  bool have_out = false;
  double* h_x[kSlots] = {};             // pinned staging for pageable callers (lazy)
  double* h_out[kSlots] = {};
  size_t cap_hx = 0;
  // small-batch path (lazy): host-mapped x and F the kernel reads and writes
  // over PCIe directly, so a small call is one launch and one sync
  static constexpr size_t kSmallValues = size_t(1) << 20;  // capacity, doubles
  size_t small_limit = kSmallValues;  // n*(k+1) <= this takes the path (profiles/r01_small_path.txt)
  double* hs_x = nullptr;
  double* hs_out = nullptr;
  double* ds_x = nullptr;
  double* ds_out = nullptr;

  int init(int dev) {
    device = dev;
    for (int s = 0; s < kSlots; ++s) {
      CUDA_TRY(cudaStreamCreateWithFlags(&stream[s], cudaStreamNonBlocking));
      CUDA_TRY(cudaEventCreateWithFlags(&copied[s], cudaEventDisableTiming));
    }
    CUDA_TRY(cudaMalloc(&d_ctr, kSlots * sizeof(unsigned long long)));
    size_t chunk = kChunkOutBytes;
    if (const char* e = std::getenv("BOYSFN_CHUNK_MB"))  // A/B experiments
      chunk = std::max<size_t>(1, std::strtoull(e, nullptr, 10)) << 20;
    cap_out = chunk / sizeof(double);
    return BOYSFN_OK;
  }

  // Device chunk buffers for chunks of cx x: the output slots once, the x
  // slots sized to cx (grown if a later call needs more; every earlier call
  // has synchronised its streams before returning).
  int ensure_chunks(size_t cx) {
    if (!have_out) {
      for (int s = 0; s < kSlots; ++s) CUDA_TRY(cudaMalloc(&d_out[s], cap_out * sizeof(double)));
      have_out = true;
    }
    if (cap_x < cx) {
      for (int s = 0; s < kSlots; ++s) {
        CUDA_TRY(cudaFree(d_x[s]));
        d_x[s] = nullptr;
        CUDA_TRY(cudaMalloc(&d_x[s], cx * sizeof(double)));
      }
      cap_x = cx;
    }
    return BOYSFN_OK;
  }

  Pipeline() = default;
  Pipeline(const Pipeline&) = delete;
  Pipeline& operator=(const Pipeline&) = delete;
  // Released when the owning host thread exits (errors ignored: at process
  // exit the runtime may already be gone).
  ~Pipeline() {
    for (int s = 0; s < kSlots; ++s) {
      if (stream[s]) cudaStreamSynchronize(stream[s]);
      cudaFree(d_x[s]);
      cudaFree(d_out[s]);
      cudaFreeHost(h_x[s]);
      cudaFreeHost(h_out[s]);
      if (copied[s]) cudaEventDestroy(copied[s]);
      if (stream[s]) cudaStreamDestroy(stream[s]);
    }
    cudaFree(d_ctr);
    cudaFreeHost(hs_x);
    cudaFreeHost(hs_out);
  }

  int ensure_small() {
    if (hs_x != nullptr) return BOYSFN_OK;
    CUDA_TRY(cudaHostAlloc(&hs_x, kSmallValues * sizeof(double), cudaHostAllocMapped));
    CUDA_TRY(cudaHostAlloc(&hs_out, kSmallValues * sizeof(double), cudaHostAllocMapped));
    CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ds_x), hs_x, 0));
    CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ds_out), hs_out, 0));
    return BOYSFN_OK;
  }

  // Pinned host staging for pageable callers: x slots of cx, output slots of
  // the chunk size.
  int ensure_staging(size_t cx) {
    if (cap_hx < cx) {
      for (int s = 0; s < kSlots; ++s) {
        CUDA_TRY(cudaFreeHost(h_x[s]));
        h_x[s] = nullptr;
        CUDA_TRY(cudaHostAlloc(&h_x[s], cx * sizeof(double), cudaHostAllocDefault));
      }
      cap_hx = cx;
    }
    for (int s = 0; s < kSlots; ++s)
      if (h_out[s] == nullptr) CUDA_TRY(cudaHostAlloc(&h_out[s], cap_out * sizeof(double), cudaHostAllocDefault));
    return BOYSFN_OK;
  }
};

// Pipelines per device, shared by every host thread: a call takes a free one
// (creating it while fewer than the bound exist) and gives it back when it
// returns, so N concurrent callers hold at most the bound's worth of device
// and pinned memory (a drop-in boys_batch_many called from 64 OpenMP threads
// would otherwise reserve 64 pipelines).  Further callers wait for a free
// pipeline; they share one PCIe link anyway.  BOYSFN_MAX_PIPELINES overrides
// the bound.  Never destroyed: at process exit the CUDA runtime may already
// be gone.
class PipelinePool {
 public:
  static PipelinePool& get() {
    static PipelinePool* pool = new PipelinePool;
    return *pool;
  }
  int acquire(int dev, Pipeline** out) {
    std::unique_lock<std::mutex> lk(mu_);
    auto& d = devs_[dev];
    cv_.wait(lk, [&] { return !d.free.empty() || d.count < bound_; });
    if (!d.free.empty()) {
      *out = d.free.back();
      d.free.pop_back();
      return BOYSFN_OK;
    }
    ++d.count;  // reserve the slot, build outside the lock
    lk.unlock();
    auto* p = new Pipeline;
    const int st = p->init(dev);
    if (st != BOYSFN_OK) {
      delete p;
      lk.lock();
      --d.count;
      cv_.notify_one();
      return st;
    }
    *out = p;
    return BOYSFN_OK;
  }
  void release(Pipeline* p) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      devs_[p->device].free.push_back(p);
    }
    cv_.notify_one();
  }
  int bound() const { return bound_; }

 private:
  PipelinePool() {
    if (const char* e = std::getenv("BOYSFN_MAX_PIPELINES")) bound_ = std::max(1, std::atoi(e));
  }
  struct PerDevice {
    std::vector<Pipeline*> free;
    int count = 0;
  };
  std::mutex mu_;
  std::condition_variable cv_;
  std::map<int, PerDevice> devs_;
  int bound_ = 4;
};

// A pipeline of the calling thread's current device for the duration of one call.
class PipelineLease {
 public:
  PipelineLease() = default;
  PipelineLease(const PipelineLease&) = delete;
  PipelineLease& operator=(const PipelineLease&) = delete;
  ~PipelineLease() {
    if (p_ != nullptr) PipelinePool::get().release(p_);
  }
  int acquire() {
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    return PipelinePool::get().acquire(dev, &p_);
  }
  Pipeline* get() const { return p_; }

 private:
  Pipeline* p_ = nullptr;
};

// Page-locked (or registered) host memory can be DMA'd directly; pageable
// memory goes through the pipeline's pinned staging instead of the driver's
// single-threaded internal staging (which ran at 10-18 GB/s on the B200 hosts).
bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

// Host-side copy of staged rows to the caller's pageable buffer, split over
// up to 16 threads (host memcpy: ~15 GB/s on 1 core, 59 on 8, 75 on 16 on the
// B200 hosts, tools/probe_hostmem.py; PCIe delivers ~55 GB/s).
struct Segment {
  double* dst;        // nullptr: check only
  const double* src;
  size_t n;
  bool check = false;  // check_input on src (first bad index -> bad)
  size_t bad = ~size_t(0);
};

// check_input (eval.cpp:13-15) as a predicate: finite and non-negative.
inline bool x_ok(double x) { return std::isfinite(x) && x >= 0; }

// First index in src[0, n) that fails x_ok, or n: blocks of 256 tested
// branch-free (vectorisable), the failing block rescanned.
size_t first_bad_x(const double* src, size_t n) {
  constexpr size_t B = 256;
  size_t i = 0;
  for (; i + B <= n; i += B) {
    bool ok = true;
    for (size_t j = 0; j < B; ++j) {
      const double v = src[i + j];
      ok &= (v >= 0.0) & (v <= 1.7976931348623157e308);
    }
    if (!ok) break;
  }
  for (; i < n; ++i)
    if (!x_ok(src[i])) return i;
  return n;
}

// Host copy of staged rows into the caller's buffer with non-temporal
// (streaming) 16-B stores: the destination is written once and never read
// back by this library, so the stores bypass the cache and skip the
// read-for-ownership of every destination line -- a quarter of the host
// memory traffic of the staged path (DMA write + copy read + copy write, no
// RFO read).  BOYSFN_COPY_NT=0 falls back to memcpy (A/B).
void copy_nt(double* dst, const double* src, size_t n) {
  static const bool nt = [] {
    const char* e = std::getenv("BOYSFN_COPY_NT");
    return !(e != nullptr && e[0] == '0');
  }();
  if (!nt || n < 64) {
    std::memcpy(dst, src, n * sizeof(double));
    return;
  }
  size_t i = 0;
  if (reinterpret_cast<uintptr_t>(dst) & 15) {  // doubles are 8-B aligned: one scalar to reach 16 B
    dst[0] = src[0];
    i = 1;
  }
  for (; i + 8 <= n; i += 8) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 2));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 4));
    const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 6));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 2), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 4), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 6), d);
  }
  for (; i < n; ++i) dst[i] = src[i];
  _mm_sfence();
}

// Persistent host-copy workers: spawning 15 threads per chunk cost ~0.3 ms
// against a ~3.7 ms copy of 128 MB.  One process-wide pool; concurrent callers
// (one staging pipeline per host thread) take turns, since they share the
// host memory bandwidth anyway.
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool pool;
    return pool;
  }
  // Runs every piece, on the calling thread plus up to T-1 workers.
  void run(std::vector<Segment>& pieces, int T) {
    std::lock_guard<std::mutex> turn(turn_mu_);
    ensure_workers(T - 1);
    {
      std::lock_guard<std::mutex> lk(mu_);
      pieces_ = &pieces;
      next_.store(0);
      helpers_ = std::min<int>(T - 1, static_cast<int>(workers_.size()));
      busy_ = helpers_;
      ++generation_;
    }
    cv_.notify_all();
    drain();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return busy_ == 0; });
    pieces_ = nullptr;
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }

 private:
  static void run_piece(Segment& s) {
    if (s.check) {
      const size_t b = first_bad_x(s.src, s.n);
      s.bad = b < s.n ? b : ~size_t(0);
      if (s.dst != nullptr) copy_nt(s.dst, s.src, b);  // rows from the first bad x on are never used
    } else {
      copy_nt(s.dst, s.src, s.n);
    }
  }
  void drain() {
    std::vector<Segment>& p = *pieces_;
    for (size_t i = next_.fetch_add(1); i < p.size(); i = next_.fetch_add(1)) run_piece(p[i]);
  }
  void ensure_workers(int want) {
    while (static_cast<int>(workers_.size()) < want) {
      const int id = static_cast<int>(workers_.size());
      workers_.emplace_back([this, id] { loop(id); });
    }
  }
  void loop(int id) {
    unsigned long long seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || (generation_ != seen && id < helpers_); });
        if (stop_) return;
        seen = generation_;
      }
      drain();
      std::lock_guard<std::mutex> lk(mu_);
      if (--busy_ == 0) done_cv_.notify_all();
    }
  }
  std::mutex turn_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  std::vector<std::thread> workers_;
  std::vector<Segment>* pieces_ = nullptr;
  std::atomic<size_t> next_{0};
  unsigned long long generation_ = 0;
  int helpers_ = 0, busy_ = 0;
  bool stop_ = false;
};

void parallel_copy(std::vector<Segment> segs) {
  size_t total = 0;
  for (const auto& g : segs) total += g.n;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int T = static_cast<int>(std::min<size_t>({16, hw, std::max<size_t>(1, total / (1u << 18))}));
  // cut the segments into pieces of about total/T doubles
  std::vector<Segment> pieces;
  const size_t piece = std::max<size_t>(1, (total + T - 1) / T);
  for (const auto& g : segs)
    for (size_t o = 0; o < g.n; o += piece) pieces.push_back({g.dst + o, g.src + o, std::min(piece, g.n - o)});
  if (T <= 1) {
    for (const auto& pc : pieces) copy_nt(pc.dst, pc.src, pc.n);
    return;
  }
  if (std::getenv("BOYSFN_COPY_SPAWN") != nullptr) {  // A/B experiments: threads per call
    std::atomic<size_t> next{0};
    auto work = [&] {
      for (size_t i = next.fetch_add(1); i < pieces.size(); i = next.fetch_add(1))
        std::memcpy(pieces[i].dst, pieces[i].src, pieces[i].n * sizeof(double));
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
    return;
  }
  CopyPool::get().run(pieces, T);
}

// check_input over xs[0, n) on the copy pool, staging the checked x into
// dst (pinned) when dst is non-null.  Returns the first bad index, or n.
// (Single-threaded, this pass bounded the host API at low k: 1e8 x at k = 8
// is 800 MB of x against 7.2 GB of F.)
size_t parallel_check_stage(double* dst, const double* xs, size_t n) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int T = static_cast<int>(std::min<size_t>({16, hw, std::max<size_t>(1, n / (1u << 17))}));
  if (T <= 1) {
    const size_t b = first_bad_x(xs, n);
    if (dst != nullptr) copy_nt(dst, xs, b);
    return b;
  }
  std::vector<Segment> pieces;
  const size_t piece = (n + T - 1) / T;
  for (size_t o = 0; o < n; o += piece) {
    Segment s{dst != nullptr ? dst + o : nullptr, xs + o, std::min(piece, n - o)};
    s.check = true;
    pieces.push_back(s);
  }
  CopyPool::get().run(pieces, T);
  for (size_t i = 0; i < pieces.size(); ++i)
    if (pieces[i].bad != ~size_t(0)) return i * piece + pieces[i].bad;
  return n;
}

// NVTX range for timeline tools (Nsight Systems): the host API's phases.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Devices a large boysfn_eval_host call is spread over (boysfn_set_devices,
// else BOYSFN_DEVICES="0,1,..."; empty = the caller's current device only).
std::mutex g_host_dev_mu;
std::vector<int> g_host_devs;
bool g_host_devs_init = false;

std::vector<int> host_devices() {
  std::lock_guard<std::mutex> lk(g_host_dev_mu);
  if (!g_host_devs_init) {
    g_host_devs_init = true;
    if (const char* e = std::getenv("BOYSFN_DEVICES")) {
      std::string v(e);
      size_t pos = 0;
      while (pos < v.size()) {
        const size_t c = v.find(',', pos);
        const std::string tok = v.substr(pos, c == std::string::npos ? std::string::npos : c - pos);
        if (!tok.empty()) g_host_devs.push_back(std::atoi(tok.c_str()));
        if (c == std::string::npos) break;
        pos = c + 1;
      }
    }
  }
  return g_host_devs;
}

// Below this many output values one device's pipeline is already at the PCIe
// link rate for most of the call; above it the shards' links add up.
constexpr size_t kMultiDeviceMinValues = size_t(1) << 24;

int eval_host_core(boysfn_tables_t t, const double* xs, size_t n, int k, double* out, size_t out_extent,
                   int layout, size_t ld, size_t* first_bad);
int eval_host_multi(boysfn_tables_t t, const double* xs, size_t n, int k, double* out, int layout, size_t ld,
                    size_t* first_bad);

}  // namespace

// ------------------------------------------------------------------ C ABI --
BOYSFN_API int boysfn_abi_version(void) { return BOYSFN_ABI_VERSION; }

BOYSFN_API const char* boysfn_status_string(int status) {
  switch (status) {
    case BOYSFN_OK: return "ok";
    case BOYSFN_ERR_SIZE: return "invalid_argument: output size mismatch";
    case BOYSFN_ERR_DOMAIN: return "domain_error: x must be finite and non-negative";
    case BOYSFN_ERR_RANGE: return "out_of_range: k outside [0, k_max]";
    case BOYSFN_ERR_TABLES: return "invalid_argument: invalid coefficient table set";
    case BOYSFN_ERR_CUDA: return "CUDA error";
    case BOYSFN_ERR_ARG: return "invalid argument";
    case BOYSFN_ERR_UNSUPPORTED: return "unsupported by the device kernels";
    case BOYSFN_ERR_INVALID: return "invalid_argument";
    default: return "unknown status";
  }
}

BOYSFN_API const char* boysfn_last_error(void) { return t_last_error.c_str(); }

BOYSFN_API int boysfn_tables_create(const boysfn_table_desc* desc, boysfn_tables_t* out) {
  if (desc == nullptr || out == nullptr) return fail(BOYSFN_ERR_ARG, "null argument");
  if (int st = check_device_desc(desc)) return st;
  auto* h = new boysfn_tables_s;
  build_handle(desc, h);
  h->valid_status = validate_desc(desc);
  if (h->valid_status != BOYSFN_OK) h->valid_msg = boysfn_last_error();
  t_last_error.clear();
  *out = h;
  return BOYSFN_OK;
}

BOYSFN_API int boysfn_tables_validate(const boysfn_table_desc* desc) {
  if (desc == nullptr) return fail(BOYSFN_ERR_ARG, "null argument");
  return validate_desc(desc);
}

BOYSFN_API int boysfn_tables_embedded(boysfn_tables_t* out) {
  if (out == nullptr) return fail(BOYSFN_ERR_ARG, "null argument");
  *out = embedded_handle();
  return BOYSFN_OK;
}

BOYSFN_API int boysfn_tables_destroy(boysfn_tables_t t) {
  if (t != nullptr && !t->is_embedded) delete t;
  return BOYSFN_OK;
}

BOYSFN_API int boysfn_tables_info(boysfn_tables_t t, double* x0, double* x1, int* k_max,
                                  double* eps_tol) {
  if (t == nullptr) return fail(BOYSFN_ERR_ARG, "null handle");
  if (x0) *x0 = t->x0;
  if (x1) *x1 = t->x1;
  if (k_max) *k_max = t->k_max;
  if (eps_tol) *eps_tol = t->eps_tol;
  return BOYSFN_OK;
}

BOYSFN_API int boysfn_eval_device(boysfn_tables_t t, const double* d_x, size_t n, int k,
                                  double* d_out, size_t out_len, int layout, size_t ld, void* stream,
                                  unsigned long long* d_first_bad) {
  if (t == nullptr) return fail(BOYSFN_ERR_ARG, "null handle");
  if (k < 0 || k > t->k_max) return fail(BOYSFN_ERR_RANGE, kMsgRange);
  if (layout != BOYSFN_LAYOUT_AOS && layout != BOYSFN_LAYOUT_SOA)
    return fail(BOYSFN_ERR_ARG, "layout must be AOS or SOA");
  if (n == 0) return BOYSFN_OK;
  if (d_x == nullptr || d_out == nullptr) return fail(BOYSFN_ERR_ARG, "null buffer");
  if (layout == BOYSFN_LAYOUT_SOA && ld < n) return fail(BOYSFN_ERR_ARG, "SOA ld must be >= n");
  const size_t need = layout == BOYSFN_LAYOUT_AOS ? n * (static_cast<size_t>(k) + 1) : static_cast<size_t>(k) * ld + n;
  if (out_len < need) return fail(BOYSFN_ERR_SIZE, kMsgSize);
  return launch_eval(t, d_x, n, k, d_out, layout, ld, static_cast<cudaStream_t>(stream),
                     d_first_bad);
}

BOYSFN_API int boysfn_eval_host(boysfn_tables_t t, const double* xs, size_t n, int k, double* out,
                                size_t out_len, int layout, size_t ld, size_t* first_bad) {
  if (t == nullptr) return fail(BOYSFN_ERR_ARG, "null handle");
  if (layout != BOYSFN_LAYOUT_AOS && layout != BOYSFN_LAYOUT_SOA)
    return fail(BOYSFN_ERR_ARG, "layout must be AOS or SOA");
  // eval.cpp:90-91: size check first (k+1 computed in size_t, as the reference).
  const size_t row = static_cast<size_t>(k) + 1;
  if (layout == BOYSFN_LAYOUT_AOS) {
    if (out_len != n * row) return fail(BOYSFN_ERR_SIZE, kMsgSize);
    ld = n;
  } else {
    if (ld < n) return fail(BOYSFN_ERR_ARG, "SOA ld must be >= n");
    if (out_len != ld * row) return fail(BOYSFN_ERR_SIZE, kMsgSize);
  }
  if (n == 0) return BOYSFN_OK;
  if (xs == nullptr || out == nullptr) return fail(BOYSFN_ERR_ARG, "null buffer");
  // check_input (eval.cpp:13-18) at the first row: x before k.
  if (k < 0 || k > t->k_max) {
    if (first_bad) *first_bad = 0;
    return x_ok(xs[0]) ? fail(BOYSFN_ERR_RANGE, kMsgRange) : fail(BOYSFN_ERR_DOMAIN, kMsgDomain);
  }
  if (host_devices().size() > 1 && n * row >= kMultiDeviceMinValues)
    return eval_host_multi(t, xs, n, k, out, layout, ld, first_bad);
  return eval_host_core(t, xs, n, k, out, layout == BOYSFN_LAYOUT_AOS ? n * row : (row - 1) * ld + n, layout, ld,
                        first_bad);
}

namespace {

// The host API on the calling thread's current device, after validation:
// out_extent = doubles from `out` the call may touch.
int eval_host_core(boysfn_tables_t t, const double* xs, size_t n, int k, double* out, size_t out_extent,
                   int layout, size_t ld, size_t* first_bad) {
  const NvtxRange range("boysfn_eval_host");
  const size_t row = static_cast<size_t>(k) + 1;
  const size_t out_len = out_extent;
  PipelineLease lease;
  if (int st = lease.acquire()) return st;
  Pipeline* P = lease.get();
  if (const char* e = std::getenv("BOYSFN_SMALL_VALUES"))  // A/B experiments
    P->small_limit = std::min<size_t>(Pipeline::kSmallValues, std::strtoull(e, nullptr, 10));
  if (n * row <= P->small_limit && std::getenv("BOYSFN_NO_SMALL_PATH") == nullptr) {
    // small batch: x and F cross PCIe inside the kernel (host-mapped pinned
    // buffers, per-warp LSU loads/stores), one launch, one synchronisation
    if (int st = P->ensure_small()) return st;
    // check_input (eval.cpp:13-15) on the host: the first bad x bounds the rows
    size_t bad = n;
    for (size_t i = 0; i < n; ++i) {
      P->hs_x[i] = xs[i];
      if (bad == n && !x_ok(xs[i])) bad = i;
    }
    const int store = layout == BOYSFN_LAYOUT_SOA ? boysfn_dev::kStoreSoA : boysfn_dev::kStoreAoSXpose;
    if (int st = launch_eval(t, P->ds_x, n, k, P->ds_out, layout, n, P->stream[0], nullptr, P->d_ctr, store))
      return st;
    CUDA_TRY(cudaStreamSynchronize(P->stream[0]));
    const size_t rows = bad;
    if (layout == BOYSFN_LAYOUT_AOS) {
      std::memcpy(out, P->hs_out, rows * row * sizeof(double));
    } else {
      for (size_t l = 0; l < row; ++l) std::memcpy(out + l * ld, P->hs_out + l * n, rows * sizeof(double));
    }
    if (bad != n) {
      if (first_bad) *first_bad = bad;
      return fail(BOYSFN_ERR_DOMAIN, kMsgDomain);
    }
    return BOYSFN_OK;
  }
  // chunks of cx x (a multiple of 32): about 1/16 of the batch's output, at
  // least 8 MB and at most the output slot (256 MB), so a mid-size batch still
  // overlaps its H2D, kernel and D2H across chunks (n = 1e6, k = 8: 2.6 -> 2.0
  // ms; n = 1e7: 16.4 -> 13.6 ms; profiles/r02_e2e_chunk.txt) while large ones
  // keep the 256-MB chunks (fewer per-chunk costs, profiles/r01_e2e_chunk.txt)
  const size_t want_out = std::min(P->cap_out, std::max<size_t>(size_t(1) << 20, n * row / 16));
  const size_t cx = std::max<size_t>(32, std::min(want_out / row, (n + 31) / 32 * 32) / 32 * 32);
  const size_t nchunks = (n + cx - 1) / cx;
  const int S = Pipeline::kSlots;
  const bool x_direct = is_pinned(xs) && is_pinned(xs + n - 1);
  const bool out_direct = is_pinned(out) && is_pinned(out + out_len - 1);
  if (int st = P->ensure_chunks(cx)) return st;
  if (!(x_direct && out_direct))
    if (int st = P->ensure_staging(cx)) return st;

  // Chunk c in slot s = c % S, all on stream s: (stage x) -> H2D -> kernel ->
  // D2H of the rows before the first bad x -> event.  x is checked on the host
  // (check_input, eval.cpp:13-15) as the chunk is issued, while earlier chunks
  // are moving, so a chunk's D2H is enqueued right behind its kernel: no
  // device flag, no host round trip, nothing small queued ahead of the big
  // copies.  (The earlier flag-and-wait scheme reached 51.5 GB/s D2H.)
  const bool soa_d2h_2d = std::getenv("BOYSFN_SOA_D2H_2D") != nullptr;  // A/B experiments
  auto issue = [&](size_t c, size_t rows) -> int {
    const NvtxRange chunk_range("boysfn chunk");
    const int s = static_cast<int>(c % S);
    const size_t off = c * cx, cn = std::min(cx, n - off);
    const double* src = x_direct ? xs + off : P->h_x[s];
    CUDA_TRY(cudaMemcpyAsync(P->d_x[s], src, cn * sizeof(double), cudaMemcpyHostToDevice, P->stream[s]));
    if (int st = launch_eval(t, P->d_x[s], cn, k, P->d_out[s], layout, cn, P->stream[s], nullptr, P->d_ctr + s))
      return st;
    if (rows > 0) {
      if (layout == BOYSFN_LAYOUT_AOS) {
        double* dst = out_direct ? out + off * row : P->h_out[s];
        CUDA_TRY(cudaMemcpyAsync(dst, P->d_out[s], rows * row * sizeof(double), cudaMemcpyDeviceToHost,
                                 P->stream[s]));
      } else if (out_direct) {
        // one 1D copy per order row (a strided 2D copy of the same rows was slower)
        if (soa_d2h_2d) {
          CUDA_TRY(cudaMemcpy2DAsync(out + off, ld * sizeof(double), P->d_out[s], cn * sizeof(double),
                                     rows * sizeof(double), row, cudaMemcpyDeviceToHost, P->stream[s]));
        } else {
          for (size_t l = 0; l < row; ++l)
            CUDA_TRY(cudaMemcpyAsync(out + l * ld + off, P->d_out[s] + l * cn, rows * sizeof(double),
                                     cudaMemcpyDeviceToHost, P->stream[s]));
        }
      } else {
        CUDA_TRY(cudaMemcpyAsync(P->h_out[s], P->d_out[s], row * cn * sizeof(double), cudaMemcpyDeviceToHost,
                                 P->stream[s]));
      }
    }
    CUDA_TRY(cudaEventRecord(P->copied[s], P->stream[s]));
    return BOYSFN_OK;
  };
  // Staged output: staging -> the caller's pageable rows, on the copy pool.
  auto unstage = [&](size_t c, size_t rows) {
    const NvtxRange unstage_range("boysfn unstage");
    const int s = static_cast<int>(c % S);
    const size_t off = c * cx, cn = std::min(cx, n - off);
    if (rows == 0) return;
    std::vector<Segment> segs;
    if (layout == BOYSFN_LAYOUT_AOS)
      segs.push_back({out + off * row, P->h_out[s], rows * row});
    else
      for (size_t l = 0; l < row; ++l) segs.push_back({out + l * ld + off, P->h_out[s] + l * cn, rows});
    parallel_copy(std::move(segs));
  };

  const bool trace = std::getenv("BOYSFN_TRACE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  auto stamp = [&](const char* what, size_t c) {
    if (trace)
      std::fprintf(stderr, "[eval_host] %8.3f ms %s %zu\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(), what, c);
  };
  int status = BOYSFN_OK;
  size_t bad_at = n;
  std::vector<std::pair<size_t, size_t>> inflight;  // (chunk, rows) whose slot may hold host staging
  const bool host_staging = !(x_direct && out_direct);
  auto retire = [&](size_t i) -> int {  // wait for inflight[i]'s copies, then move its staged rows out
    const auto [c, rows] = inflight[i];
    if (cudaError_t e = cudaEventSynchronize(P->copied[c % S])) return cuda_fail(e, "cudaEventSynchronize");
    if (!out_direct) unstage(c, rows);
    stamp("retired", c);
    return BOYSFN_OK;
  };
  size_t head = 0;  // first inflight entry not yet retired
  for (size_t c = 0; c < nchunks; ++c) {
    const int s = static_cast<int>(c % S);
    const size_t off = c * cx, cn = std::min(cx, n - off);
    if (host_staging && c >= static_cast<size_t>(S)) {  // the slot's staging buffers come back
      if ((status = retire(head++))) break;
    }
    // x check (and pageable staging) of this chunk, on the copy pool
    const size_t b = off + parallel_check_stage(x_direct ? nullptr : P->h_x[s], xs + off, cn);
    const size_t rows = b - off;
    if ((status = issue(c, rows))) break;
    stamp("issued", c);
    inflight.emplace_back(c, rows);
    if (rows < cn) {
      bad_at = b;
      break;
    }
  }
  while (host_staging && head < inflight.size()) {
    const int st = retire(head++);
    if (status == BOYSFN_OK) status = st;
  }
  for (int s = 0; s < S; ++s) cudaStreamSynchronize(P->stream[s]);
  if (status == BOYSFN_OK) {
    if (cudaError_t e = cudaGetLastError()) return cuda_fail(e, "boysfn_eval_host");
    if (bad_at != n) {
      if (first_bad) *first_bad = bad_at;
      return fail(BOYSFN_ERR_DOMAIN, kMsgDomain);
    }
  }
  return status;
}

// One persistent host thread per listed device (so each keeps its staging
// pipeline), running one shard of a multi-device boysfn_eval_host call.
class DeviceWorker {
 public:
  explicit DeviceWorker(int device) : device_(device), th_([this] { loop(); }) {}
  ~DeviceWorker() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    th_.join();
  }
  void submit(std::function<void()> job) {
    std::lock_guard<std::mutex> lk(mu_);
    job_ = std::move(job);
    done_ = false;
    cv_.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return done_; });
  }

 private:
  void loop() {
    cudaSetDevice(device_);
    for (;;) {
      std::function<void()> job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || job_ != nullptr; });
        if (stop_) return;
        job = std::move(job_);
        job_ = nullptr;
      }
      job();
      std::lock_guard<std::mutex> lk(mu_);
      done_ = true;
      cv_.notify_all();
    }
  }
  int device_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::function<void()> job_;
  bool done_ = true, stop_ = false;
  std::thread th_;  // last: started after the members it uses
};

// Splits [0, n) over the listed devices (x checked on the host first: rows
// from the first bad x on are never written, as eval.cpp:92-95).  Each shard
// is a single-device call on its worker; the caller gets the first failure.
int eval_host_multi(boysfn_tables_t t, const double* xs, size_t n, int k, double* out, int layout, size_t ld,
                    size_t* first_bad) {
  const NvtxRange range("boysfn_eval_host multi-device");
  static std::mutex multi_mu;  // one multi-device call at a time (the workers are shared)
  std::lock_guard<std::mutex> lk(multi_mu);
  static std::map<std::pair<size_t, int>, std::unique_ptr<DeviceWorker>> workers;  // (list position, device)
  const std::vector<int> devs = host_devices();
  const size_t row = static_cast<size_t>(k) + 1;
  // first bad x, on the copy pool's threads
  const int T = static_cast<int>(std::min<unsigned>(16, std::max(1u, std::thread::hardware_concurrency())));
  std::vector<size_t> bad(T, n);
  {
    std::vector<std::thread> th;
    for (int i = 0; i < T; ++i)
      th.emplace_back([&, i] {
        const size_t a = n * i / T, b = n * (i + 1) / T;
        for (size_t j = a; j < b; ++j)
          if (!x_ok(xs[j])) {
            bad[i] = j;
            break;
          }
      });
    for (auto& h : th) h.join();
  }
  const size_t neff = *std::min_element(bad.begin(), bad.end());
  const size_t D = devs.size();
  std::vector<int> status(D, BOYSFN_OK);
  std::vector<std::string> msg(D);
  for (size_t d = 0; d < D; ++d) {
    const size_t a = neff * d / D, b = neff * (d + 1) / D;
    auto& w = workers[{d, devs[d]}];
    if (!w) w = std::make_unique<DeviceWorker>(devs[d]);
    if (b == a) continue;
    w->submit([&, d, a, b] {
      double* o = layout == BOYSFN_LAYOUT_AOS ? out + a * row : out + a;
      const size_t extent = layout == BOYSFN_LAYOUT_AOS ? (b - a) * row : (row - 1) * ld + (b - a);
      status[d] = eval_host_core(t, xs + a, b - a, k, o, extent, layout, ld, nullptr);
      if (status[d] != BOYSFN_OK) msg[d] = boysfn_last_error();
    });
  }
  for (size_t d = 0; d < D; ++d) {
    const size_t a = neff * d / D, b = neff * (d + 1) / D;
    if (b > a) workers[{d, devs[d]}]->wait();
  }
  for (size_t d = 0; d < D; ++d)
    if (status[d] != BOYSFN_OK) return fail(status[d], "device " + std::to_string(devs[d]) + ": " + msg[d]);
  if (neff != n) {
    if (first_bad) *first_bad = neff;
    return fail(BOYSFN_ERR_DOMAIN, kMsgDomain);
  }
  return BOYSFN_OK;
}

}  // namespace

BOYSFN_API int boysfn_host_alloc(size_t bytes, void** ptr) {
  if (ptr == nullptr) return fail(BOYSFN_ERR_ARG, "null argument");
  *ptr = nullptr;
  if (bytes == 0) return BOYSFN_OK;
  CUDA_TRY(cudaHostAlloc(ptr, bytes, cudaHostAllocPortable));  // pinned for every device
  return BOYSFN_OK;
}

BOYSFN_API int boysfn_host_free(void* ptr) {
  if (ptr != nullptr) CUDA_TRY(cudaFreeHost(ptr));
  return BOYSFN_OK;
}

BOYSFN_API int boysfn_set_devices(const int* devices, int count) {
  if (count > 0 && devices == nullptr) return fail(BOYSFN_ERR_ARG, "null device list");
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  for (int i = 0; i < count; ++i)
    if (devices[i] < 0 || devices[i] >= ndev) return fail(BOYSFN_ERR_ARG, "no such device");
  std::lock_guard<std::mutex> lk(g_host_dev_mu);
  g_host_devs.assign(devices, devices + std::max(count, 0));
  g_host_devs_init = true;
  return BOYSFN_OK;
}

BOYSFN_API int boysfn_eval_region_host(boysfn_tables_t t, double x, int k, int region, double* out) {
  if (t == nullptr || out == nullptr) return fail(BOYSFN_ERR_ARG, "null argument");
  if (region < 0 || region > 2) return fail(BOYSFN_ERR_ARG, "region must be A, B or C");
  if (!x_ok(x)) return fail(BOYSFN_ERR_DOMAIN, kMsgDomain);
  if (k < 0 || k > t->k_max) return fail(BOYSFN_ERR_RANGE, kMsgRange);
  if (region == BOYSFN_REGION_B && !(x > 0)) return fail(BOYSFN_ERR_DOMAIN, kMsgUpward);
  if (!t->degree_ok[k]) return fail(BOYSFN_ERR_UNSUPPORTED, "table degree exceeds the device image (max 23)");
  if (k > BOYSFN_DEVICE_KMAX_RT)
    return fail(BOYSFN_ERR_UNSUPPORTED, "order above the run-time-k kernels' bound (64)");
  PipelineLease lease;
  if (int st = lease.acquire()) return st;
  Pipeline* P = lease.get();
  // one x in, one row out, through the host-mapped small-call buffers
  if (int st = P->ensure_small()) return st;
  cudaStream_t s = P->stream[0];
  P->hs_x[0] = x;
  if (k > boysfn_dev::kKernelKmax) {
    if (int st = launch_generic(t, P->ds_x, 1, k, P->ds_out, BOYSFN_LAYOUT_AOS, 1, s, nullptr, region, P->d_ctr,
                                false))
      return st;
  } else {
    EvalParams p = t->params[k];
    void* args[] = {&p, &x, &region, &P->ds_out};
    CUDA_TRY(cudaLaunchKernel(boysfn_dev::kernel_region(k, t->variant[k]), dim3(1), dim3(1), args, 0, s));
    boysfn_internal::count_launch();
  }
  CUDA_TRY(cudaStreamSynchronize(s));
  std::memcpy(out, P->hs_out, (k + 1) * sizeof(double));
  return BOYSFN_OK;
}

// -------------------------------------------------------- workload gens --
namespace {

__device__ __forceinline__ double uniform01(uint64_t seed, uint64_t idx) {
  uint64_t z = seed + (idx + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return static_cast<double>(z >> 11) * 0x1.0p-53;
}

__global__ void gen_uniform_kernel(double* x, size_t n, uint64_t seed, uint64_t offset, double lo,
                                   double span) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    x[i] = __dadd_rn(lo, __dmul_rn(span, uniform01(seed, offset + i)));
}

__global__ void gen_loguniform_kernel(double* x, size_t n, uint64_t seed, uint64_t offset, double lo,
                                      double span) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    x[i] = exp10(__dadd_rn(lo, __dmul_rn(span, uniform01(seed, offset + i))));
}

// configs[2] boundary stress: each x independently
// picks a breakpoint b in {0+, x0, x1} and a mode -- b +- j ulps (|j| <= 64),
// b +- 10^-s with s ~ U[1,15], or b + U[-1,1] -- then |.|; keyed by the global
// index, so consecutive x (one warp) mix regions like a shuffled batch.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void gen_boundary_kernel(double* x, size_t n, uint64_t seed, uint64_t offset, double x0, double x1) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const uint64_t z = mix64(seed + (offset + i + 1) * 0x9E3779B97F4A7C15ull);
    const uint64_t w = mix64(z ^ 0xD1B54A32D192ED03ull);
    const int which = static_cast<int>(z % 3), mode = static_cast<int>((z >> 8) % 3);
    const double u = static_cast<double>(w >> 11) * 0x1.0p-53;
    const double b = which == 0 ? 0.0 : which == 1 ? x0 : x1;
    double v;
    if (mode == 0) {
      const long long j = static_cast<long long>((w >> 20) % 129) - 64;
      v = b == 0.0 ? static_cast<double>(j < 0 ? -j : j) * 4.9406564584124654e-324
                   : __longlong_as_double(__double_as_longlong(b) + j);
    } else if (mode == 1) {
      const double off = exp10(-(1.0 + 14.0 * u));
      v = ((w >> 10) & 1) ? b + off : b - off;
    } else {
      v = b + (2.0 * u - 1.0);
    }
    x[i] = fabs(v);
  }
}

int gen_grid(size_t n, unsigned* grid) {
  int dev = 0, sms = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  *grid = static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>((n + 255) / 256, size_t(sms) * 8)));
  return BOYSFN_OK;
}

}  // namespace

BOYSFN_API int boysfn_generate_uniform(double* d_x, size_t n, uint64_t seed, uint64_t offset,
                                       double lo, double hi, void* stream) {
  if (n == 0) return BOYSFN_OK;
  if (d_x == nullptr) return fail(BOYSFN_ERR_ARG, "null buffer");
  unsigned grid = 0;
  if (int st = gen_grid(n, &grid)) return st;
  gen_uniform_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(d_x, n, seed, offset, lo, hi - lo);
  CUDA_TRY(cudaGetLastError());
  boysfn_internal::count_launch();
  return BOYSFN_OK;
}

BOYSFN_API int boysfn_generate_loguniform(double* d_x, size_t n, uint64_t seed, uint64_t offset,
                                          double log10_lo, double log10_hi, void* stream) {
  if (n == 0) return BOYSFN_OK;
  if (d_x == nullptr) return fail(BOYSFN_ERR_ARG, "null buffer");
  unsigned grid = 0;
  if (int st = gen_grid(n, &grid)) return st;
  gen_loguniform_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(d_x, n, seed, offset, log10_lo,
                                                                             log10_hi - log10_lo);
  CUDA_TRY(cudaGetLastError());
  boysfn_internal::count_launch();
  return BOYSFN_OK;
}

BOYSFN_API int boysfn_generate_boundary(double* d_x, size_t n, uint64_t seed, uint64_t offset, double x0,
                                        double x1, void* stream) {
  if (n == 0) return BOYSFN_OK;
  if (d_x == nullptr) return fail(BOYSFN_ERR_ARG, "null buffer");
  unsigned grid = 0;
  if (int st = gen_grid(n, &grid)) return st;
  gen_boundary_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(d_x, n, seed, offset, x0, x1);
  CUDA_TRY(cudaGetLastError());
  boysfn_internal::count_launch();
  return BOYSFN_OK;
}

BOYSFN_API unsigned long long boysfn_kernel_launch_count(void) {
  return g_launches.load(std::memory_order_relaxed);
}

// Exact degrees of the embedded kernels (boys_launch.h).
void boysfn_dev::embedded_degrees(int k, int* na, int* ma, int* nb, int* mb) {
  *na = (k >= 0 && k <= BOYSFN_EMB_KMAX) ? kEmbDegA[k][0] : -1;
  *ma = (k >= 0 && k <= BOYSFN_EMB_KMAX) ? kEmbDegA[k][1] : -1;
  *nb = kEmbDegB[0];
  *mb = kEmbDegB[1];
}
