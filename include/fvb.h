/*
 * fvb.h -- C ABI of the B200-native evaluation backend (libfvb.so).
 *
 * This is the drop-in boundary for the hot path of the fusevec reference
 * (arXiv 1809.09851, FDBB/UETLI): fused single-pass evaluation of vector
 * expressions and compressible-flow building blocks over long
 * structure-of-arrays vectors.  Plain pointers and sizes only; no C++ types,
 * no exceptions cross it.  Every entry point returns an fvb_status;
 * fvb_last_error() gives the message of the calling thread's last failure.
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   - the runtime-JIT C ABI `detail::JitKernel::Fn`
 *       void(size_t begin, size_t end, void* const* args)   src/jit.hpp:14-17
 *     obtained from `jit_kernel_for(const Expr&, Precision)` src/jit.hpp:22
 *     with the argument block of `jit_args`                 src/jit.hpp:24-29
 *     -> fvb_kernel / fvb_lookup below (same argument-block convention:
 *        outputs first, then one slot per distinct leaf in first-appearance
 *        DFS order; device pointers; async on a CUDA stream);
 *   - the per-item evaluation loop of `evaluate`            src/backend_eval.cpp:280-346
 *     and `evaluate_block` / `eval_block_core`              src/block.cpp:373-463
 *     -> one fused multi-output kernel per block expression (fvb_flux,
 *        fvb_cons2prim, fvb_jacobian, ...);
 *   - the reference's fluid expression objects evaluated through them
 *       inviscid_flux     src/fluid.cpp:273-310   -> fvb_flux
 *       convert/derived_p src/fluid.cpp:234-271   -> fvb_cons2prim, fvb_prim2cons
 *       derived_v_mag2    src/fluid.cpp:243-247   -> fvb_v_mag2
 *       eos_ideal_p/_T    src/fluid.cpp:57-65     -> fvb_eos
 *     plus the blocks the reference lacks: sound
 *     speed (in fvb_cons2prim), flux Jacobians and the CFL max wave speed
 *     (fvb_jacobian, fvb_wave_speed_max).
 *
 * Conventions
 *   - Precision codes match fusevec::Precision (include/fusevec/
 *     dense_vector.hpp:17): 0 = f32, 1 = f64.  Every plane of one call has
 *     the call's precision; arithmetic happens in that precision with every
 *     constant narrowed first, exactly as the reference evaluates an all-f32
 *     or all-f64 tree (src/scalar_ops.hpp:83-85, src/expr.cpp:109).
 *   - A d-dimensional conservative state is d+2 planes in canonical order
 *     [rho, m_0 .. m_{d-1}, rhoE]; a primitive state [rho, v_0.., p].
 *     Block outputs are row-major item lists (include/fusevec/block.hpp:14-17).
 *   - Device entry points take DEVICE pointers and enqueue on `stream`
 *     (a cudaStream_t; NULL = the legacy default stream).  They never
 *     synchronise.  n == 0 is a no-op that returns FVB_OK.
 *   - Aliasing.  The named entry points (fvb_flux, fvb_cons2prim, ...)
 *     reject, with FVB_EARG before any launch, an output plane that is an
 *     input plane; fvb_axpy_sin is the exception (y is in/out, as the
 *     reference lets dest alias a leaf, backend.hpp:44-46).  Kernels from
 *     fvb_lookup accept an output that IS a leaf plane (in-place evaluation,
 *     as JitKernel::Fn does) and then read with coherent loads.  A block
 *     kernel computes every item from the planes as they were at launch; the
 *     reference's item-by-item loop (block.cpp:413-451) differs only when an
 *     item reads a plane an earlier item writes, and the C++ adapter
 *     evaluates such blocks item by item.  Every entry point rejects planes
 *     that overlap at an offset.  Two outputs may name one plane: the later
 *     item's value is stored last.
 *   - Results are bitwise identical to the reference for +,-,*,/,sqrt;
 *     sin differs by at most CUDA's 2-ulp bound from glibc's.
 */
#ifndef FVB_H
#define FVB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FVB_ABI_VERSION 1

/* Only the entry points below are exported from libfvb.so (it is built
 * with -fvisibility=hidden). */
#if defined(__GNUC__)
#define FVB_API __attribute__((visibility("default")))
#else
#define FVB_API
#endif

typedef enum fvb_status {
    FVB_OK = 0,
    FVB_ELEN = 1,         /* length mismatch (fusevec::LengthMismatch)           */
    FVB_EPREC = 2,        /* unsupported precision code                          */
    FVB_ECUDA = 3,        /* CUDA runtime error (launch, copy, allocation)       */
    FVB_ENCCL = 4,        /* collective failure (reserved for the host runtime)  */
    FVB_EARG = 5,         /* bad argument: NULL plane, dim out of range, ...     */
    FVB_EUNSUPPORTED = 6, /* no kernel for this structural key                   */
    FVB_EALIGN = 7,       /* a plane pointer is not element-aligned              */
    FVB_EHOST = 8         /* host-side failure: memory, threads (no exception    */
                          /* ever crosses this ABI)                              */
} fvb_status;

typedef enum fvb_prec { FVB_F32 = 0, FVB_F64 = 1 } fvb_prec;

/* Ideal-gas constants as the reference derives them from EosSpec
 * (include/fusevec/fluid.hpp:27-45, src/fluid.cpp:40-53):
 * gamma_minus_one = (R/cv).value(), gamma = (cp/cv).value(), cv = cv.value().
 * NULL everywhere means the default diatomic gas cp=7/2, cv=5/2. */
typedef struct fvb_gas {
    double gamma_minus_one;
    double gamma;
    double cv;
} fvb_gas;

/* ---- library ------------------------------------------------------------ */

FVB_API int fvb_abi_version(void);
/* Message for the calling thread's last non-OK status ("" if none). */
FVB_API const char* fvb_last_error(void);
/* Human-readable build description (arch, flags). */
FVB_API const char* fvb_build_info(void);

/* ---- device-pointer entry points (async on `stream`) --------------------- */

/* y <- 0.5*sin(x+y), in place (paper Fig. 2; proj/tests/test_backend.cpp:41). */
FVB_API fvb_status fvb_axpy_sin(uint8_t prec, uint64_t n, const void* x, void* y, void* stream);

/* Inviscid flux F(U) of a conservative state, all d directions in one pass
 * (src/fluid.cpp:273-310).  in: d+2 planes; out: (d+2)*d planes, item r*d+c. */
FVB_API fvb_status fvb_flux(const fvb_gas* gas, uint32_t dim, uint8_t prec, uint64_t n,
                    const void* const* in, void* const* out, void* stream);

/* Inviscid flux of a PRIMITIVE state [rho, v_0..v_{d-1}, p]
 * (src/fluid.cpp:290-298): same (d+2)*d item layout as fvb_flux. */
FVB_API fvb_status fvb_flux_prim(const fvb_gas* gas, uint32_t dim, uint8_t prec, uint64_t n,
                                 const void* const* in, void* const* out, void* stream);

/* Conservative -> primitive + EOS in one pass (src/fluid.cpp:234-258 and
 * SURVEY A.2): in: d+2 planes; out: d+2 planes [v_0..v_{d-1}, p, c].
 * rho passes through (the reference's convert reuses the density node). */
FVB_API fvb_status fvb_cons2prim(const fvb_gas* gas, uint32_t dim, uint8_t prec, uint64_t n,
                         const void* const* in, void* const* out, void* stream);

/* Primitive -> conservative (src/fluid.cpp:259-268): in [rho, v.., p];
 * out d+1 planes [m_0..m_{d-1}, rhoE]. */
FVB_API fvb_status fvb_prim2cons(const fvb_gas* gas, uint32_t dim, uint8_t prec, uint64_t n,
                         const void* const* in, void* const* out, void* stream);

/* derived_v_mag2 of a conservative state (src/fluid.cpp:243-247), the
 * paper's micro-benchmark (mx^2+my^2+mz^2)/rho^2.  Reads in[0..d] (rho and
 * the momenta; rhoE is not touched), out: one plane. */
FVB_API fvb_status fvb_v_mag2(uint32_t dim, uint8_t prec, uint64_t n, const void* const* in,
                      void* out, void* stream);

/* Ideal-gas closures (src/fluid.cpp:57-65): p = gm1*(rho*e), T = e/cv.
 * Either output may be NULL. */
FVB_API fvb_status fvb_eos(const fvb_gas* gas, uint8_t prec, uint64_t n, const void* rho,
                   const void* e, void* p, void* T, void* stream);

/* Flux Jacobians A_k = dF_k/dU, k < d, dense (d+2)x(d+2) each, layout
 * [k][r][c] (d*(d+2)^2 planes), fused with the CFL wave-speed
 * maximum lambda_max = max_i sqrt(v_mag2_i) + c_i (A.4).  lambda_max is a
 * DEVICE scalar of the call's precision (or NULL to skip the reduction); it
 * is overwritten (not accumulated) in stream order.  NaN if any lambda is
 * NaN; 0 for n == 0. */
FVB_API fvb_status fvb_jacobian(const fvb_gas* gas, uint32_t dim, uint8_t prec, uint64_t n,
                        const void* const* in, void* const* out, void* lambda_max,
                        void* stream);

/* Read-only CFL pass: lambda_max only (A.4); same semantics as above.
 * lambda (optional, may be NULL) receives the per-point wave speed. */
FVB_API fvb_status fvb_wave_speed_max(const fvb_gas* gas, uint32_t dim, uint8_t prec, uint64_t n,
                              const void* const* in, void* lambda, void* lambda_max,
                              void* stream);

/* CSR sparse matrix-vector accumulation of the block layer (paper Eq. 2;
 * csr_matvec_acc, src/block.cpp:345-357): y[r] += sum_k (TY)v[k]*(TY)x[ci[k]]
 * for r < rows, the row's nonzeros summed in stored order in y's precision
 * (bitwise the reference's order).  row_ptr (rows+1 entries), col_idx and
 * values (nnz entries, already narrowed to the matrix precision as
 * SparseMatrix stores them) are DEVICE arrays; x and y device planes of
 * precisions prec_x / prec_y.  The arrays must form a valid CSR matrix, as
 * SparseMatrix guarantees (row_ptr non-decreasing from 0 to nnz, every
 * column index inside x): the device does not re-check the structure.
 * NULL or misaligned arrays are refused (FVB_EARG / FVB_EALIGN). */
FVB_API fvb_status fvb_csr_matvec_acc(uint8_t prec_y, uint8_t prec_x, uint64_t rows, uint64_t nnz,
                                      const uint64_t* row_ptr, const uint64_t* col_idx,
                                      const double* values, const void* x, void* y,
                                      void* stream);

/* The same with 32-bit column indices (any matrix with fewer than 2^32
 * columns): the device-resident layout the C++ adapter's DeviceCsr keeps,
 * 12 instead of 16 bytes per nonzero of index + value stream.  The
 * reference stores size_t indices (SparseMatrix, block.hpp:42-44); the
 * narrowing happens once, at upload, and changes no result bit. */
FVB_API fvb_status fvb_csr_matvec_acc_u32(uint8_t prec_y, uint8_t prec_x, uint64_t rows,
                                          uint64_t nnz, const uint64_t* row_ptr,
                                          const uint32_t* col_idx, const double* values,
                                          const void* x, void* y, void* stream);

/* On-device synthetic inputs, bit-identical to the reference's host
 * generators because SplitMix64 is random-access (proj/include/fusevec/
 * rng.hpp:8-28):
 *  - fvb_synth_state: the random_state of proj/tests/acceptance.cpp:214-230
 *    for global points [first, first+n) -> d+2 conservative planes (an f32
 *    call stores the f64 value narrowed, as DenseVector::set does);
 *  - fvb_synth_uniform: make_vec of proj/tests/oracle.hpp:118-123, element
 *    t = uniform(lo, hi) of draw first+t. */
FVB_API fvb_status fvb_synth_state(uint32_t dim, uint8_t prec, uint64_t seed, uint64_t first,
                           uint64_t n, void* const* out, void* stream);
FVB_API fvb_status fvb_synth_uniform(uint8_t prec, uint64_t seed, uint64_t first, uint64_t n,
                             double lo, double hi, void* out, void* stream);

/* ---- JitKernel-shaped lookup (src/jit.hpp:12-29) ------------------------- */

/* A kernel found by structural key: a closure over the constants and the
 * leaf-slot permutation captured from the key.  Launch it as
 *     k.fn(&k, begin, end, args, stream)
 * with args = [outputs (row-major items)..., one slot per distinct leaf in
 * first-appearance DFS order] as DEVICE pointers -- the argument block of
 * jit_args (src/jit.hpp:24-29, src/backend_jit.cpp:78-99, 337-345) -- and
 * [begin, end) the element range, like JitKernel::Fn. */
typedef struct fvb_kernel fvb_kernel;
typedef fvb_status (*fvb_kernel_fn)(const fvb_kernel* self, uint64_t begin, uint64_t end,
                                    void* const* args, void* stream);
/* For blocks that carry a CFL wave speed (Jacobian, wave speed): the same
 * pass, additionally max-accumulating lambda over [begin, end) into the
 * DEVICE scalar lambda_max (of the kernel's precision).  It accumulates --
 * the caller zeroes it once -- so a range split into chunks reduces to the
 * same value.  For the wave-speed block args[0] may be NULL (reduce only). */
typedef fvb_status (*fvb_kernel_reduce_fn)(const fvb_kernel* self, uint64_t begin, uint64_t end,
                                           void* const* args, void* lambda_max, void* stream);

struct fvb_kernel {
    fvb_kernel_fn fn;
    fvb_kernel_reduce_fn reduce; /* NULL unless the block has a CFL reduction */
    uint32_t n_outputs;  /* leading output slots in args                      */
    uint32_t n_inputs;   /* distinct leaf slots after them                    */
    uint32_t n_consts;   /* valid entries of consts                           */
    uint8_t prec;        /* precision of every slot (0 f32, 1 f64)            */
    uint8_t dim;         /* spatial dimension of a fluid block (0 otherwise)  */
    int8_t in_slot[8];   /* canonical input i is args[n_outputs + in_slot[i]];
                            all -1 for a lowered kernel (no canonical order)  */
    double consts[8];    /* captured constants, named per kernel  */
    char name[48];       /* e.g. "flux3_f64", or "gen:<hash>" when lowered    */
    const void* impl;    /* opaque: the NVRTC-lowered kernel, else NULL       */
};

/* Resolve a structural key.  Single expressions use the reference's own
 * key grammar verbatim (dest precision char + key_node of the tree,
 * src/backend_jit.cpp:112-155, 319-322); fused block expressions use
 * "G<rows>x<cols>:" followed by one such key per item with leaf slots
 * numbered across the whole block.
 *
 * A key matching a hand-written fused kernel returns it, with the key's
 * constants captured into out->consts.  Any other well-formed key is lowered
 * -- the B200 counterpart of the reference's runtime JIT
 * (src/backend_jit.cpp:179-335) -- into one CUDA kernel: every item of the
 * block computed per element with common subexpressions shared across
 * items, each node in its own precision with operands converted first and
 * constants as exact hex literals (the reference's emit / emit_as rules),
 * compiled by NVRTC for sm_100a with --fmad=false and cached per key for
 * the process lifetime (and the compiled image on disk under
 * $FVB_CACHE_DIR, default ~/.cache/fvb, keyed by the exact source and NVRTC
 * version; FVB_CACHE_DIR=off disables it).  FVB_EUNSUPPORTED for a
 * malformed key, a non-finite constant or when NVRTC is unavailable;
 * FVB_ECUDA when the compiled kernel cannot be loaded (no device). */
FVB_API fvb_status fvb_lookup(const char* key, fvb_kernel* out);

/* The CUDA source fvb_lookup would compile for `key` (NUL-terminated into
 * buf when it fits; *len receives the full length).  Pure host code. */
FVB_API fvb_status fvb_emit_source(const char* key, char* buf, size_t cap, size_t* len);

/* Compile `key`'s lowered kernel with NVRTC without loading it (no GPU
 * needed); *cubin_bytes receives the sm_100a image size. */
FVB_API fvb_status fvb_nvrtc_compile(const char* key, size_t* cubin_bytes);

/* Number of registered patterns and the i-th pattern (a constant written
 * "C<p>#<name>;" is a wildcard captured into consts under that name; every
 * occurrence of one name must carry the same bits), for diagnostics and
 * tests. */
FVB_API uint32_t fvb_pattern_count(void);
FVB_API const char* fvb_pattern(uint32_t i, const char** name);

/* ---- host-buffer entry points (the end-to-end path) ---------------------- */

/* A per-device context owning staging buffers and copy/compute streams for
 * the host-buffer entry points.  chunk_points = points per pipeline stage
 * (0 = as many as fit 256 MiB of device staging per slot).  Not thread-safe:
 * one call at a time per context. */
typedef struct fvb_ctx fvb_ctx;
FVB_API fvb_status fvb_ctx_create(int device, uint64_t chunk_points, fvb_ctx** out);
FVB_API fvb_status fvb_ctx_destroy(fvb_ctx* ctx);

/* Same operation as fvb_flux / fvb_jacobian, but `in` and `out` are HOST
 * pointers (pinned or pageable).  The range is streamed through the device
 * in chunks with host->device copies, the fused kernel and device->host
 * copies overlapped on separate streams; returns after the last byte is
 * back in host memory.  lambda_max is a HOST double.  A device pointer
 * among the host planes is refused (FVB_EARG), and so is a host plane that
 * is not element-aligned (FVB_EALIGN), before anything runs. */
FVB_API fvb_status fvb_flux_host(fvb_ctx* ctx, const fvb_gas* gas, uint32_t dim, uint8_t prec,
                         uint64_t n, const void* const* in, void* const* out);
FVB_API fvb_status fvb_jacobian_host(fvb_ctx* ctx, const fvb_gas* gas, uint32_t dim, uint8_t prec,
                             uint64_t n, const void* const* in, void* const* out,
                             double* lambda_max);

/* Any structural-key kernel (fvb_lookup) over HOST arrays: the staged
 * executor behind the two calls above, for the C++ adapter's host
 * DenseVectors.  args is the kernel's argument block (k->n_outputs outputs,
 * then k->n_inputs leaves in slot order); arg_prec[i] is 0 (f32) or 1 (f64);
 * arg_on_device[i] = 1 marks a DEVICE plane used in place, 2 an output the
 * caller does not want back (computed into device scratch only, e.g. a
 * pass-through item the caller copies host-side); NULL = all host.
 * Host planes may be pinned or pageable: pageable ones are packed into
 * pinned bounce buffers by host threads, overlapped with the device work.
 * An output may be one of the host leaves (in-place evaluation); a NULL
 * output slot is allowed where the kernel allows it.  With lambda_max
 * (HOST double) the kernel's CFL reduction runs as well.  Device work
 * already queued on `after` (a cudaStream_t, may be NULL) completes before
 * the call reads any plane.  Returns once every output is in place. */
FVB_API fvb_status fvb_launch_host(fvb_ctx* ctx, const fvb_kernel* k, uint64_t n,
                                   void* const* args, const uint8_t* arg_prec,
                                   const uint8_t* arg_on_device, double* lambda_max,
                                   void* after);

#ifdef __cplusplus
}
#endif

#endif /* FVB_H */
