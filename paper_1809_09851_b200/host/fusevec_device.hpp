// fusevec_device.hpp -- the B200 device backend behind the reference's own
// C++ API (proj/include/fusevec/backend.hpp, block.hpp, fluid.hpp).
//
// This is the host-side half of the drop-in: it compiles against the
// reference's public headers, takes the reference's Expr / BlockExpr /
// StateSet objects unchanged, computes the same structural key the
// reference's JIT cache uses (proj/src/backend_jit.cpp:112-155), resolves it
// to a fused sm_100a kernel through the C ABI (include/fvb.h: fvb_lookup), and
// launches it with the reference's argument-block convention (jit_args,
// proj/src/jit.hpp:24-29).  It adds the pieces the north_star names that the
// reference lacks: a device-resident vector (make_temp), multi-output
// destinations (tie), the sound-speed / Jacobian / wave-speed expression
// objects and the CFL maximum.
//
// Integration: the reference gains BackendKind::Device and
// forwards evaluate / evaluate_block to the functions below.  Until then a
// caller passes a DeviceBackend explicitly.  No CPU fallback exists: an
// expression with no fused kernel throws UnsupportedExpression.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

#include "fusevec/backend.hpp"
#include "fusevec/bench.hpp"
#include "fusevec/block.hpp"
#include "fusevec/dense_vector.hpp"
#include "fusevec/error.hpp"
#include "fusevec/expr.hpp"
#include "fusevec/fluid.hpp"

namespace fusevec {

/// A CUDA runtime / launch failure (status FVB_ECUDA).
struct DeviceError : Error {
    using Error::Error;
};

/// The expression's structural key has no fused device kernel.
struct UnsupportedExpression : Error {
    using Error::Error;
};

// ---- new fluid expression objects, reference style ----

/// Sound speed c = sqrt((gamma*p)/rho), lazily (A.2).
Expr derived_c(const StateSet& u);

/// Wave speed lambda = sqrt(v_mag2) + c per point (A.4).
Expr wave_speed(const StateSet& u);

/// Flux Jacobians A_k = dF_k/dU of a conservative state (A.3): a
/// (d*(d+2)) x (d+2) block, item (k*(d+2)+r, c) = A_k[r][c].
BlockExpr inviscid_flux_jacobian(const StateSet& u);

namespace device {

/// Device-resident SoA plane: the storage type's device variant.  Owns a
/// cudaMalloc allocation of size() elements of precision().
class DeviceVector {
  public:
    DeviceVector() = default;
    DeviceVector(Precision prec, std::size_t len);
    ~DeviceVector();
    DeviceVector(const DeviceVector&) = delete;
    DeviceVector& operator=(const DeviceVector&) = delete;
    DeviceVector(DeviceVector&& o) noexcept;
    DeviceVector& operator=(DeviceVector&& o) noexcept;

    Precision precision() const { return prec_; }
    std::size_t size() const { return len_; }
    std::size_t byte_size() const { return len_ * scalar_width(prec_); }
    void* data() { return ptr_; }
    const void* data() const { return ptr_; }

    void upload(const DenseVector& host);     // synchronous H2D
    void download(DenseVector& host) const;  // synchronous D2H

  private:
    Precision prec_ = Precision::f64;
    std::size_t len_ = 0;
    void* ptr_ = nullptr;
};

/// UETLI make_temp: a device temporary of the given precision and length.
DeviceVector make_temp(Precision prec, std::size_t len);

/// Binds host DenseVector leaves to device-resident copies: expressions
/// whose leaves are bound read the device planes and move no host memory.
/// A SparseMatrix's CSR arrays uploaded once (row pointers, column indices
/// and the stored values, block.hpp:42-44), for repeated block matvecs
/// without re-sending the matrix over PCIe.  A snapshot: re-upload after
/// SparseMatrix::set_value.  Column indices are kept as 32-bit integers
/// when the matrix has fewer than 2^32 columns (12 instead of 16 streamed
/// bytes per nonzero; no result bit changes), else as the reference's
/// 64-bit size_t.
class DeviceCsr {
  public:
    explicit DeviceCsr(const SparseMatrix& m, int ordinal = 0);
    ~DeviceCsr();
    DeviceCsr(const DeviceCsr&) = delete;
    DeviceCsr& operator=(const DeviceCsr&) = delete;

    void upload(const SparseMatrix& m);  // refresh from the host matrix
    std::size_t rows() const { return rows_; }
    std::size_t cols() const { return cols_; }
    std::size_t nnz() const { return nnz_; }
    const std::uint64_t* row_ptr() const { return rp_; }
    /// true: col_idx32() holds the indices; false: col_idx() does
    bool narrow_indices() const { return narrow_; }
    const std::uint64_t* col_idx() const { return narrow_ ? nullptr : static_cast<const std::uint64_t*>(ci_); }
    const std::uint32_t* col_idx32() const { return narrow_ ? static_cast<const std::uint32_t*>(ci_) : nullptr; }
    const double* values() const { return v_; }

  private:
    int ordinal_ = 0;
    std::size_t rows_ = 0, cols_ = 0, nnz_ = 0;
    bool narrow_ = false;
    std::uint64_t* rp_ = nullptr;
    void* ci_ = nullptr;
    double* v_ = nullptr;
};

class Residency {
  public:
    Residency();
    Residency(const Residency& o);
    Residency& operator=(const Residency& o);

    void bind(const DenseVector& host, DeviceVector& dev);
    void unbind(const DenseVector& host);
    DeviceVector* find(const DenseVector* host) const;
    /// Block matvecs with this matrix read the device copy.
    void bind(const SparseMatrix& host, DeviceCsr& dev);
    void unbind(const SparseMatrix& host);
    DeviceCsr* find(const SparseMatrix* host) const;

    /// Changes with every bind / unbind and is unique per object (copies
    /// get their own): evaluations that reuse one block expression key
    /// their cached launch plan on it.
    std::uint64_t version() const { return version_; }

  private:
    std::unordered_map<const DenseVector*, DeviceVector*> map_;
    std::unordered_map<const SparseMatrix*, DeviceCsr*> csr_;
    std::uint64_t version_;
};

/// Evaluation strategy for the device path (the analog of Backend).
struct DeviceBackend {
    int ordinal = 0;
    void* stream = nullptr;              // cudaStream_t; nullptr = legacy default
    const Residency* residency = nullptr;
    std::size_t chunk_points = 0;  // host-buffer staging chunk (0 = 256 MiB of device staging per slot)
    /// Host-buffer evaluations (every plane a host vector) may spread over
    /// several devices: the range is cut into one contiguous slice per
    /// ordinal, each streamed over its own PCIe link in parallel, and the CFL
    /// maxima combined exactly.  Empty = `ordinal` alone.
    std::vector<int> ordinals;
    /// false: an evaluation whose planes are all on the device returns once
    /// its kernel is enqueued on `stream` (no host wait), so a sequence of
    /// evaluate / evaluate_block calls can overlap, or be captured into a
    /// CUDA graph and replayed.  Calls that return a value (the CFL maxima)
    /// and host-buffer evaluations always complete before returning.
    bool synchronize = true;
};

/// UETLI tie: a list of device destinations a multi-output block writes in
/// one pass (row-major item order).
struct Tie {
    std::vector<DeviceVector*> dests;
};
template <class... Ds>
Tie tie(Ds&... ds) {
    return Tie{{&ds...}};
}

/// The reference's structural key of e for a destination of precision dest
/// (backend_jit.cpp:112-155, 319-322); "" if a constant is non-finite.
std::string structural_key(const Expr& e, Precision dest);

/// Fused block key: "G<r>x<c>:" + per-item keys joined by
/// '|', leaf slots numbered across the block; `leaves` receives the slots.
std::string block_key(const std::vector<Expr>& items, const std::vector<Precision>& dests,
                      std::size_t rows, std::size_t cols,
                      std::vector<const DenseVector*>* leaves);

/// dest[i] = e[i] on the device.  Host leaves/destination are staged through
/// the device in chunks; bound (resident) ones are used in place.
void evaluate(const DeviceBackend& be, const Expr& e, DenseVector& dest);
void evaluate(const DeviceBackend& be, const Expr& e, DeviceVector& dest);

/// All items of a block in one fused pass (the reference evaluates them one
/// by one: proj/src/block.cpp:373-451).
void evaluate_block(const DeviceBackend& be, const BlockExpr& e, BlockVectorGrid& dest);
void evaluate_block(const DeviceBackend& be, const BlockExpr& e, BlockColVector& dest);
void evaluate_block(const DeviceBackend& be, const BlockExpr& e, const Tie& dest);

/// CFL maximum of a per-point wave-speed expression (wave_speed(u)):
/// one fused device reduction, exact.  NaN if any lambda is NaN; 0 if empty.
double reduce_max(const DeviceBackend& be, const Expr& lambda);

/// Jacobian block fused with the CFL reduction: writes the block and returns
/// max_i lambda_i of the same state in the same pass.
double evaluate_block_cfl(const DeviceBackend& be, const BlockExpr& jacobian,
                          BlockVectorGrid& dest);
double evaluate_block_cfl(const DeviceBackend& be, const BlockExpr& jacobian, const Tie& dest);
/// The same, leaving the maximum on the device in lambda_max (one element of
/// the block's precision) instead of returning it: no host read-back, so with
/// synchronize = false a time loop's Jacobian + CFL step can be captured in
/// a CUDA graph and the maximum consumed by later device work.
void evaluate_block_cfl(const DeviceBackend& be, const BlockExpr& jacobian, const Tie& dest,
                        DeviceVector& lambda_max);

// ---- the reference's benchmark harness on the device (fusevec_device_bench.cpp) ----

/// Where the benchmark's planes live: device-resident (leaves bound through
/// a Residency, outputs DeviceVectors / a Tie) or the reference's own host
/// DenseVectors (staged over PCIe on every call).
enum class BenchPlanes { Device, Host };

/// Backend label of device records: "b200x<G>" (G = ordinals, at least 1).
std::string bench_label(const DeviceBackend& be);

/// proj/include/fusevec/bench.hpp run_micro / run_miniapp with the device
/// backend: cfg's suite, sizes, reps, precision as the reference reads them
/// (cfg.backend is ignored: `be` evaluates).  Records carry the same fields;
/// overhead_ratio = the reference-API call (evaluate / evaluate_block of the
/// reference's tree) over the fused kernel called directly through the C ABI.
/// Throws OracleMismatch if either differs from the other or from the
/// reference's Backend::scalar_ref() in one bit.  write_csv (bench.hpp)
/// writes the records in the reference's CSV schema.
std::vector<BenchRecord> run_micro(const BenchConfig& cfg, const DeviceBackend& be,
                                   BenchPlanes where = BenchPlanes::Device);
std::vector<BenchRecord> run_miniapp(const BenchConfig& cfg, const DeviceBackend& be,
                                     BenchPlanes where = BenchPlanes::Device);

}  // namespace device
}  // namespace fusevec
