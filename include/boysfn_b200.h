/*
 * boysfn_b200.h -- C ABI of the B200-native batched Boys-function evaluator.
 *
 * This is the drop-in boundary for the reference hot path
 *   void boysfn::boys_batch_many(std::span<const double> xs, int k,
 *                                const boysfn::CoefficientTableSet& tables,
 *                                std::span<double> out);
 * (/root/reference/proj/core/include/boysfn/eval.hpp:43-45, implemented at
 *  /root/reference/proj/core/src/eval.cpp:88-96).  The reference has no FFI of
 * its own; this header is what a binding (cgo / JNI / ctypes / the C++ shim in
 * paper_2512_10059_b200/cpp/) links against.  Plain C types only: no
 * exceptions cross it, every entry point returns a boysfn_status, streams are
 * passed as opaque cudaStream_t handles (void*; NULL = legacy default stream).
 *
 * Thread safety: table handles are immutable after creation and may be shared
 * across threads and streams; concurrent calls on different streams are safe.
 */
#ifndef BOYSFN_B200_H
#define BOYSFN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BOYSFN_ABI_VERSION 2  /* 2: boysfn_eval_device takes out_len */

/* Error convention.  The reference throws C++ exceptions; each maps to one code
 * and the C++ shim rethrows the same type with the same message. */
typedef enum boysfn_status {
  BOYSFN_OK = 0,
  BOYSFN_ERR_SIZE = 1,        /* std::invalid_argument, eval.cpp:90-91            */
  BOYSFN_ERR_DOMAIN = 2,      /* std::domain_error, x < 0 or non-finite, eval.cpp:14-15 */
  BOYSFN_ERR_RANGE = 3,       /* std::out_of_range, k outside [0, k_max], eval.cpp:16-17 */
  BOYSFN_ERR_TABLES = 4,      /* std::invalid_argument from validate_tables, tables.cpp:14-32 */
  BOYSFN_ERR_CUDA = 5,        /* a CUDA runtime error (no reference equivalent)   */
  BOYSFN_ERR_ARG = 6,         /* NULL handle/pointer or bad layout/ld             */
  BOYSFN_ERR_UNSUPPORTED = 7, /* a table degree beyond the device image (or Algorithm 2 with k > 32) */
  BOYSFN_ERR_INVALID = 8      /* other std::invalid_argument (verify_tables arguments, verify.cpp:15-18) */
} boysfn_status;

/* Output layout.  AOS is the reference's row-major out[i*(k+1)+l]
 * (eval.cpp:94); SOA (out[l*ld+i]) is a north-star addition. */
typedef enum boysfn_layout { BOYSFN_LAYOUT_AOS = 0, BOYSFN_LAYOUT_SOA = 1 } boysfn_layout;

/* Region seam, boysfn::Region (eval.hpp:17). */
typedef enum boysfn_region { BOYSFN_REGION_A = 0, BOYSFN_REGION_B = 1, BOYSFN_REGION_C = 2 } boysfn_region;

/* Flattened boysfn::RationalApproximant (tables.hpp:12-17): ascending degree,
 * numer has n+1 and denom m+1 entries, denom[m] == 1 (monic). */
typedef struct boysfn_rational_desc {
  int n;
  int m;
  const double* numer;
  const double* denom;
} boysfn_rational_desc;

/* Flattened boysfn::CoefficientTableSet (tables.hpp:21-28). */
typedef struct boysfn_table_desc {
  double x0;
  double x1;
  int k_max;
  double eps_tol;
  boysfn_rational_desc r_B;
  const boysfn_rational_desc* r_A; /* k_max + 1 entries, indexed by k */
} boysfn_table_desc;

/* Opaque immutable device-side table image built from a table set. */
typedef struct boysfn_tables_s* boysfn_tables_t;

/* Largest order of the templated (unrolled, tuned) kernels; orders above it
 * -- table sets with k_max > 32, e.g. from the reference's gen path
 * (k_max <= 64) -- run on the run-time-k generic kernel. */
#define BOYSFN_DEVICE_KMAX 32
/* Largest order any kernel evaluates (the run-time-k kernels; SPEC.md:476
 * caps generated sets at k_max <= 64).  Sets with a larger k_max load, but
 * orders above this return BOYSFN_ERR_UNSUPPORTED. */
#define BOYSFN_DEVICE_KMAX_RT 64
/* Largest numerator / denominator degree the device image holds. */
#define BOYSFN_DEVICE_MAX_DEGREE 23

int boysfn_abi_version(void);
const char* boysfn_status_string(int status);
/* Message of the last error on the calling thread (exact reference wording for
 * SIZE/DOMAIN/RANGE/TABLES, CUDA error text for CUDA). */
const char* boysfn_last_error(void);

/* Build a table handle from a table set and copy the coefficients.  Replaces
 * passing `const CoefficientTableSet&` (eval.hpp:44) across the boundary.
 * Like eval.cpp, which evaluates any set it is given, it refuses only what
 * the device image cannot hold: k_max < 0, a missing r_A array, empty or
 * non-finite coefficient vectors (BOYSFN_ERR_TABLES, validate_tables'
 * messages).  The full validate_tables outcome is recorded in the handle and
 * enforced by boysfn_verify_tables, as verify.cpp:14 does. */
int boysfn_tables_create(const boysfn_table_desc* desc, boysfn_tables_t* out);
/* validate_tables (tables.cpp:14-32): same checks, order and messages;
 * BOYSFN_ERR_TABLES with boysfn_last_error() set on the first failure. */
int boysfn_tables_validate(const boysfn_table_desc* desc);
/* Process-lifetime handle of the embedded Appendix-C set (k_max = 32,
 * eps = 5e-14), the device image of embedded_default() (tables_data.cpp:8). */
int boysfn_tables_embedded(boysfn_tables_t* out);
/* Destroying the embedded handle is a no-op. */
int boysfn_tables_destroy(boysfn_tables_t tables);
int boysfn_tables_info(boysfn_tables_t tables, double* x0, double* x1, int* k_max,
                       double* eps_tol);

/* Device entry point: x and out already resident in HBM.  Evaluates
 * F_0..F_k for all n arguments, enqueued on `stream`, asynchronous.
 *   layout AOS: out[i*(k+1)+l]  (ld ignored)   needs out_len >= n*(k+1)
 *   layout SOA: out[l*ld+i]     (ld >= n)      needs out_len >= k*ld + n
 * out_len = doubles the caller owns at d_out; a smaller value returns
 * BOYSFN_ERR_SIZE (the reference's size check, eval.cpp:90-91) and launches
 * nothing.  Any alignment and any ld are accepted (TMA stores either way).
 * Invalid x (negative, NaN, +-inf) does not stop the launch: when
 * d_first_bad is non-NULL the kernel lowers *d_first_bad (a device uint64 the
 * caller initialised, e.g. to UINT64_MAX) to the smallest offending index with
 * atomicMin; rows at and after that index are unspecified.  Returns
 * BOYSFN_ERR_RANGE for k outside [0, k_max] (host-side, nothing launched). */
int boysfn_eval_device(boysfn_tables_t tables, const double* d_x, size_t n, int k,
                       double* d_out, size_t out_len, int layout, size_t ld, void* stream,
                       unsigned long long* d_first_bad);

/* Host entry point with boys_batch_many semantics (eval.cpp:88-96): xs and out
 * are host buffers (pageable or pinned), out_len must equal n*(k+1) for AOS
 * (else BOYSFN_ERR_SIZE) or ld*(k+1) with ld >= n for SOA.  Streams the batch
 * through the device in chunks with host<->device copies overlapped with the
 * kernels, and synchronises before returning.  On a bad x the rows before it
 * are written, later rows are left untouched and *first_bad (if non-NULL)
 * receives its index, exactly like the reference's first-throw behaviour. */
int boysfn_eval_host(boysfn_tables_t tables, const double* xs, size_t n, int k, double* out,
                     size_t out_len, int layout, size_t ld, size_t* first_bad);

/* Page-locked host memory for boysfn_eval_host buffers.  Pinned x and out
 * are read and written by the copy engines directly (about 55 GB/s D2H on
 * the B200 hosts); pageable ones go through the library's pinned staging plus
 * a host memcpy (27-33 GB/s).  Callers that reuse their buffers across calls
 * should allocate them here.  *ptr = NULL for bytes == 0. */
int boysfn_host_alloc(size_t bytes, void** ptr);
int boysfn_host_free(void* ptr);

/* Spreads large boysfn_eval_host calls (n*(k+1) >= 2^24 values) over these
 * devices: contiguous shards of the batch, one persistent host thread and
 * staging pipeline per device, so the shards' PCIe links add up (the
 * reference's boys_batch_many is a single call, eval.hpp:44-45).  x is checked
 * on the host first, so the rows from the first bad x on are never written.
 * count <= 0 restores the default (the calling thread's current device); the
 * environment variable BOYSFN_DEVICES="0,1,..." sets the initial list.  A
 * device may appear more than once (tests). */
int boysfn_set_devices(const int* devices, int count);

/* Forced-region evaluation of one x (boys_batch_region, eval.cpp:59-81, the
 * reference's branch-agreement test seam), computed on the device. */
int boysfn_eval_region_host(boysfn_tables_t tables, double x, int k, int region, double* out);

/* verify_tables (verify.hpp:12-35, verify.cpp:12-63) on the device: samples
 * samples_per_region x uniformly in each region (A [0,x0), B [x0,x1),
 * C [x1,xmax]) with the reference's generator (std::mt19937_64(seed),
 * u = (rng() >> 11) * 2^-53), evaluates every order k = 0..k_max and an
 * extended-precision (double-double) oracle, and reports per (k, region) the
 * maximum |F - oracle| with the reference's worst-case bookkeeping.
 * per_k: caller array of (k_max+1)*3 doubles, [k][A, B, C]. */
typedef struct boysfn_verify_report {
  double max_err;
  double worst_x;
  int worst_k;
  char worst_region; /* 'A', 'B', 'C' or '-' */
  double max_err_region[3];
  double* per_k;
} boysfn_verify_report;
int boysfn_verify_tables(boysfn_tables_t tables, int samples_per_region, double xmax, uint64_t seed,
                         boysfn_verify_report* report);

/* Algorithm 2 of the paper, fused on the
 * device: z_i = sum_{l=0..k} c_l sum_j F_l(x_i + x_j) y_j for i < n, with
 * x, y, z device arrays of n doubles (x >= 0, finite), c a HOST array of k+1
 * doubles.  F_l are Algorithm 1's values (regions A/B/C of the table set);
 * no Boys value is stored.  Enqueued on `stream` (sort, gather, O(n^2) pair
 * kernel, scatter), asynchronous; scratch comes from the stream-ordered pool. */
int boysfn_alg2_device(boysfn_tables_t tables, const double* d_x, const double* d_y, size_t n, int k,
                       const double* c, double* d_z, void* stream);

/* Coefficient generator support (replaces the
 * grid scan and golden-section refinement of remez.cpp:33-108, ErrorCurve).
 * For HOST arrays xs[npts] writes err[i] = rho(x) (F_k(x) - p(x)/q(x)) with
 * F_k by the reference's series (reference.cpp:10-23), p and q by Horner,
 * all in double-double on the device; p, q given as double-double coefficient
 * pairs (hi, lo), ascending, degrees n, m <= 64; weight 0: rho = 1 (r_B),
 * 1: rho = rho_A,k (Eq. 18, regions.cpp:74-85).  k <= 64.  Synchronous. */
int boysfn_gen_error_scan(int k, const double* num_hi, const double* num_lo, int n, const double* den_hi,
                          const double* den_lo, int m, int weight, const double* xs, size_t npts,
                          double* err);
/* F_k(xs[i]) in double-double (hi[i] + lo[i]), HOST arrays, synchronous. */
int boysfn_gen_boys_dd(int k, const double* xs, size_t npts, double* hi, double* lo);

/* Synthetic workload: x[i] = lo + (hi-lo)*u_i with u_i = (splitmix64(seed +
 * (offset+i+1)*0x9E3779B97F4A7C15) >> 11) * 2^-53, the multiply and add
 * separately rounded, so any CPU restating the formula reproduces it bit for
 * bit and a shard [offset, offset+n) of the global stream is independent of
 * the shard count. */
int boysfn_generate_uniform(double* d_x, size_t n, uint64_t seed, uint64_t offset, double lo,
                            double hi, void* stream);
/* x[i] = 10^(log10_lo + (log10_hi-log10_lo)*u_i) (same u_i). */
int boysfn_generate_loguniform(double* d_x, size_t n, uint64_t seed, uint64_t offset,
                               double log10_lo, double log10_hi, void* stream);

/* configs[2] boundary stress: x clustered at 0+, x0 and x1 (+-j ulps with
 * |j| <= 64, +-10^-s with s ~ U[1,15], or U[b-1, b+1]), |x| taken, every x
 * keyed by its global index (so warps mix regions). */
int boysfn_generate_boundary(double* d_x, size_t n, uint64_t seed, uint64_t offset, double x0, double x1,
                             void* stream);

/* Number of this library's kernels launched by the calling process so far
 * (bench.py reports the delta over its timed region as gpu_launches). */
unsigned long long boysfn_kernel_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* BOYSFN_B200_H */
