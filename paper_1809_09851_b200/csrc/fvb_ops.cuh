// fvb_ops.cuh -- per-point arithmetic of every fused block, sm_100a.
//
// Each Op describes one block expression of the fusevec reference as a
// pointwise map from NIN input planes to NOUT output planes:
//   prepare(in, k)  -> State  : the shared subexpressions (CSE across items)
//   out(s, j, k)    -> T      : item j of the block, j a compile-time constant
//                                after unrolling, so the if-chains fold away
//   lambda(s, k)    -> T      : optional per-point wave speed (CFL reduction)
//
// Bitwise parity with the reference comes from three rules, all checked by
// the parity tests:
//   1. identical operation order and association to the reference's trees
//      (each function cites the tree it mirrors);
//   2. no FMA contraction: this file is compiled with --fmad=false (the
//      reference builds with -ffp-contract=off, proj/CMakeLists.txt:11-14);
//   3. constants arrive already narrowed to T (Consts<T>, filled on the host
//      exactly like scalar_ops.hpp:83-85 narrow_value), and every operation
//      runs in T, as an all-f32 / all-f64 tree evaluates (expr.cpp:109).
// Sharing a subexpression (v_j, p) between items is bitwise neutral: the
// reference recomputes the same operations on the same operands per item.
#pragma once

#include <cstdint>

namespace fvb {

template <class T>
struct Consts {
    T half;   // constant(0.5, ...)
    T gm1;    // gamma - 1 = (R/cv).value()      src/fluid.cpp:53
    T gamma;  // (cp/cv).value()
    T cv;     // cv.value()                      src/fluid.cpp:62-65
    T zero;   // 0 and 1 entries of the Jacobian
    T one;
};

// sum_of_squares: left-associated from the first square (src/fluid.cpp:222-230).
template <int D, class T>
__device__ __forceinline__ T sum_sq(const T (&q)[D]) {
    T acc = q[0] * q[0];
#pragma unroll
    for (int j = 1; j < D; ++j) acc = acc + q[j] * q[j];
    return acc;
}

// derived_p, conservative branch (src/fluid.cpp:234-241):
//   kin = 0.5*(msq/rho); p = gm1*(rhoE - kin)
template <class T>
__device__ __forceinline__ T pressure(const Consts<T>& k, T rho, T msq, T rho_E) {
    T kin = k.half * (msq / rho);
    return k.gm1 * (rho_E - kin);
}

// Sound speed: elem_sqrt((constant(gamma, p) * p) / rho).
template <class T>
__device__ __forceinline__ T sound_speed(const Consts<T>& k, T rho, T p) {
    return sqrt((k.gamma * p) / rho);
}

// ---------------------------------------------------------------------------
// inviscid_flux of a conservative state (src/fluid.cpp:273-310):
//   F(0,j) = m_j;  F(1+i,j) = m_i*(m_j/rho) [+ p iff i==j];
//   F(d+1,j) = (m_j/rho)*(rhoE + p);  row-major item r*d + j.
// ---------------------------------------------------------------------------
template <class T, int D>
struct FluxOp {
    static constexpr int NIN = D + 2;
    static constexpr int NOUT = (D + 2) * D;
    static constexpr bool HAS_LAMBDA = false;
    static constexpr bool ALIASED = false;
    struct State {
        T m[D], v[D], p, rho_E;
    };
    __device__ __forceinline__ static State prepare(const T (&in)[NIN], const Consts<T>& k) {
        State s;
        const T rho = in[0];
#pragma unroll
        for (int j = 0; j < D; ++j) s.m[j] = in[1 + j];
        s.rho_E = in[D + 1];
        s.p = pressure(k, rho, sum_sq<D>(s.m), s.rho_E);
#pragma unroll
        for (int j = 0; j < D; ++j) s.v[j] = s.m[j] / rho;
        return s;
    }
    __device__ __forceinline__ static T out(const State& s, int item, const Consts<T>&) {
        const int r = item / D, c = item % D;
        if (r == 0) return s.m[c];
        if (r <= D) {
            T f = s.m[r - 1] * s.v[c];
            if (r - 1 == c) f = f + s.p;
            return f;
        }
        return s.v[c] * (s.rho_E + s.p);
    }
    __device__ __forceinline__ static T lambda(const State&, const Consts<T>&) { return T(0); }
};

// ---------------------------------------------------------------------------
// inviscid_flux of a PRIMITIVE state [rho, v.., p] (src/fluid.cpp:290-298):
//   rho_v_j = rho*v_j;  rhoE = p/gm1 + 0.5*(rho*vsq);
//   F(0,j) = rho_v_j;  F(1+i,j) = rho_v_i*v_j [+ p iff i==j];
//   F(d+1,j) = v_j*(rhoE + p).
// ---------------------------------------------------------------------------
template <class T, int D>
struct FluxPrimOp {
    static constexpr int NIN = D + 2;
    static constexpr int NOUT = (D + 2) * D;
    static constexpr bool HAS_LAMBDA = false;
    static constexpr bool ALIASED = false;
    struct State {
        T rv[D], v[D], p, rho_E;
    };
    __device__ __forceinline__ static State prepare(const T (&in)[NIN], const Consts<T>& k) {
        State s;
        const T rho = in[0];
#pragma unroll
        for (int j = 0; j < D; ++j) s.v[j] = in[1 + j];
        s.p = in[D + 1];
#pragma unroll
        for (int j = 0; j < D; ++j) s.rv[j] = rho * s.v[j];
        s.rho_E = s.p / k.gm1 + k.half * (rho * sum_sq<D>(s.v));
        return s;
    }
    __device__ __forceinline__ static T out(const State& s, int item, const Consts<T>&) {
        const int r = item / D, c = item % D;
        if (r == 0) return s.rv[c];
        if (r <= D) {
            T f = s.rv[r - 1] * s.v[c];
            if (r - 1 == c) f = f + s.p;
            return f;
        }
        return s.v[c] * (s.rho_E + s.p);
    }
    __device__ __forceinline__ static T lambda(const State&, const Consts<T>&) { return T(0); }
};

// ---------------------------------------------------------------------------
// convert(u, Primitive) fields 1..d+1 (src/fluid.cpp:249-258) + sound speed:
//   out = [m_0/rho, ..., m_{d-1}/rho, p, sqrt((gamma*p)/rho)]
// ---------------------------------------------------------------------------
template <class T, int D>
struct Cons2PrimOp {
    static constexpr int NIN = D + 2;
    static constexpr int NOUT = D + 2;
    static constexpr bool HAS_LAMBDA = false;
    static constexpr bool ALIASED = false;
    struct State {
        T v[D], p, c;
    };
    __device__ __forceinline__ static State prepare(const T (&in)[NIN], const Consts<T>& k) {
        State s;
        const T rho = in[0];
        T m[D];
#pragma unroll
        for (int j = 0; j < D; ++j) m[j] = in[1 + j];
        s.p = pressure(k, rho, sum_sq<D>(m), in[D + 1]);
#pragma unroll
        for (int j = 0; j < D; ++j) s.v[j] = m[j] / rho;
        s.c = sound_speed(k, rho, s.p);
        return s;
    }
    __device__ __forceinline__ static T out(const State& s, int item, const Consts<T>&) {
        if (item < D) return s.v[item];
        return item == D ? s.p : s.c;
    }
    __device__ __forceinline__ static T lambda(const State&, const Consts<T>&) { return T(0); }
};

// ---------------------------------------------------------------------------
// convert(u, Conservative) fields 1..d+1 (src/fluid.cpp:259-268):
//   m_i = rho*v_i;  rhoE = p/gm1 + 0.5*(rho*vsq)
// ---------------------------------------------------------------------------
template <class T, int D>
struct Prim2ConsOp {
    static constexpr int NIN = D + 2;
    static constexpr int NOUT = D + 1;
    static constexpr bool HAS_LAMBDA = false;
    static constexpr bool ALIASED = false;
    struct State {
        T rho, v[D], p;
    };
    __device__ __forceinline__ static State prepare(const T (&in)[NIN], const Consts<T>&) {
        State s;
        s.rho = in[0];
#pragma unroll
        for (int j = 0; j < D; ++j) s.v[j] = in[1 + j];
        s.p = in[D + 1];
        return s;
    }
    __device__ __forceinline__ static T out(const State& s, int item, const Consts<T>& k) {
        if (item < D) return s.rho * s.v[item];
        return s.p / k.gm1 + k.half * (s.rho * sum_sq<D>(s.v));
    }
    __device__ __forceinline__ static T lambda(const State&, const Consts<T>&) { return T(0); }
};

// derived_v_mag2, conservative (src/fluid.cpp:243-247): msq/(rho*rho).
// Reads [rho, m_0..m_{d-1}] only (4R + 1W = 40 B/pt in 3-D fp64).
template <class T, int D>
struct VMag2Op {
    static constexpr int NIN = D + 1;
    static constexpr int NOUT = 1;
    static constexpr bool HAS_LAMBDA = false;
    static constexpr bool ALIASED = false;
    struct State {
        T r;
    };
    __device__ __forceinline__ static State prepare(const T (&in)[NIN], const Consts<T>&) {
        T m[D];
#pragma unroll
        for (int j = 0; j < D; ++j) m[j] = in[1 + j];
        return State{sum_sq<D>(m) / (in[0] * in[0])};
    }
    __device__ __forceinline__ static T out(const State& s, int, const Consts<T>&) { return s.r; }
    __device__ __forceinline__ static T lambda(const State&, const Consts<T>&) { return T(0); }
};

// eos_ideal_p (src/fluid.cpp:57-60): rho_e = rho*e; gm1*rho_e.
// eos_ideal_T (src/fluid.cpp:62-65): e/cv.   in = [rho, e]; out = [p, T].
template <class T, int MASK>  // bit 0: p, bit 1: T
struct EosOp {
    static constexpr int NIN = 2;
    static constexpr int NOUT = (MASK & 1) + ((MASK >> 1) & 1);
    static constexpr bool HAS_LAMBDA = false;
    static constexpr bool ALIASED = false;
    struct State {
        T rho, e;
    };
    __device__ __forceinline__ static State prepare(const T (&in)[NIN], const Consts<T>&) {
        return State{in[0], in[1]};
    }
    __device__ __forceinline__ static T out(const State& s, int item, const Consts<T>& k) {
        const bool want_p = (MASK & 1) && item == 0;
        if (want_p) return k.gm1 * (s.rho * s.e);
        return s.e / k.cv;
    }
    __device__ __forceinline__ static T lambda(const State&, const Consts<T>&) { return T(0); }
};

// ---------------------------------------------------------------------------
// Flux Jacobians A_k = dF_k/dU, layout [k][r][c], W = d+2:
//   u_j = m_j/rho; q2 = sum u_j^2; H = (rhoE+p)/rho; phi = 0.5*(gm1*q2)
//   row 0       = e_{k+1}
//   row 1+i     : c0  = i==k ? phi - u_i*u_k : -(u_i*u_k)
//                 c1+j= left-to-right sum of [u_k if i==j], [u_i if j==k],
//                       [-(gm1*u_j) if i==k], or 0
//                 cW-1= i==k ? gm1 : 0
//   row d+1     : c0  = u_k*(phi - H)
//                 c1+j= j==k ? H - gm1*(u_j*u_k) : -(gm1*(u_j*u_k))
//                 cW-1= gamma*u_k
// plus lambda = sqrt(msq/(rho*rho)) + sqrt((gamma*p)/rho) (A.4).
// ---------------------------------------------------------------------------
template <class T, int D>
struct JacobianOp {
    static constexpr int W = D + 2;
    static constexpr int NIN = D + 2;
    static constexpr int NOUT = D * W * W;
    static constexpr bool HAS_LAMBDA = true;
    static constexpr bool ALIASED = false;
    struct State {
        T u[D], H, phi, lam;
    };
    __device__ __forceinline__ static State prepare(const T (&in)[NIN], const Consts<T>& k) {
        State s;
        const T rho = in[0];
        const T rho_E = in[D + 1];
        T m[D];
#pragma unroll
        for (int j = 0; j < D; ++j) m[j] = in[1 + j];
        const T msq = sum_sq<D>(m);
        const T p = pressure(k, rho, msq, rho_E);
#pragma unroll
        for (int j = 0; j < D; ++j) s.u[j] = m[j] / rho;
        const T q2 = sum_sq<D>(s.u);
        s.H = (rho_E + p) / rho;
        s.phi = k.half * (k.gm1 * q2);
        s.lam = sqrt(msq / (rho * rho)) + sound_speed(k, rho, p);
        return s;
    }
    // The items that are constants whatever the state (30 of the 75 in 3-D:
    // row 0, the momentum rows' last column, and the momentum entries with
    // no term): their value, shared by the kernel and the host-buffer path
    // (which fills them host-side instead of shipping them over PCIe).
    __host__ __device__ __forceinline__ static bool constant_item(int item, const Consts<T>& k,
                                                                  T* v) {
        const int dir = item / (W * W);
        const int r = (item / W) % W;
        const int c = item % W;
        if (r == 0) {
            *v = c == 1 + dir ? k.one : k.zero;
            return true;
        }
        if (r <= D && c == W - 1) {
            *v = r - 1 == dir ? k.gm1 : k.zero;
            return true;
        }
        if (r <= D && c != 0 && r - 1 != c - 1 && c - 1 != dir && r - 1 != dir) {
            *v = k.zero;
            return true;
        }
        return false;
    }
    // Items computed by the same expression as an earlier item (18 of the 45
    // non-constant ones in 3-D): u_m appears four times (t0- or t1-only
    // momentum entries), -(gm1*u_m) twice, and -(u_i*u_k) and
    // -(gm1*(u_j*u_k)) once per direction of the pair (IEEE products are
    // commutative, so both orders give the same bits).  The host-buffer
    // path ships one copy over PCIe and copies it host-side.
    __host__ __device__ static int value_id(int item) {
        const int dir = item / (W * W);
        const int r = (item / W) % W;
        const int c = item % W;
        if (r >= 1 && r <= D) {
            const int i = r - 1;
            if (c >= 1 && c <= D) {
                const int j = c - 1;
                const bool t0 = (i == j), t1 = (j == dir), t2 = (i == dir);
                if (t0 && !t1 && !t2) return 16 + dir;  // u_dir
                if (t1 && !t0 && !t2) return 16 + i;    // u_i
                if (t2 && !t0 && !t1) return 32 + j;    // -(gm1*u_j)
                return -1;
            }
            if (c == 0 && i != dir) return 48 + 4 * (i < dir ? i : dir) + (i < dir ? dir : i);
            return -1;
        }
        if (r == W - 1 && c >= 1 && c <= D && c - 1 != dir) {
            const int j = c - 1;
            return 64 + 4 * (j < dir ? j : dir) + (j < dir ? dir : j);
        }
        return -1;
    }
    __host__ __device__ static int duplicate_of(int item) {
        const int id = value_id(item);
        if (id < 0) return -1;
        for (int e = 0; e < item; ++e)
            if (value_id(e) == id) return e;
        return -1;
    }
    __device__ __forceinline__ static T out(const State& s, int item, const Consts<T>& k) {
        T cv;
        if (constant_item(item, k, &cv)) return cv;
        const int dir = item / (W * W);
        const int r = (item / W) % W;
        const int c = item % W;
        const T uk = s.u[dir];
        if (r <= D) {
            const int i = r - 1;
            if (c == 0) return i == dir ? s.phi - s.u[i] * uk : -(s.u[i] * uk);
            const int j = c - 1;
            // Present terms in the fixed order of A.3 (at least one present:
            // the term-free entries are constant items).
            const bool t0 = (i == j), t1 = (j == dir), t2 = (i == dir);
            T acc;
            if (t0) acc = uk;
            if (t1) acc = t0 ? acc + s.u[i] : s.u[i];
            if (t2) {
                const T t = -(k.gm1 * s.u[j]);
                acc = (t0 || t1) ? acc + t : t;
            }
            return acc;
        }
        if (c == 0) return uk * (s.phi - s.H);
        if (c == W - 1) return k.gamma * uk;
        const int j = c - 1;
        const T ujuk = s.u[j] * uk;
        return j == dir ? s.H - k.gm1 * ujuk : -(k.gm1 * ujuk);
    }
    __device__ __forceinline__ static T lambda(const State& s, const Consts<T>&) { return s.lam; }
};

// Read-only CFL pass (A.4): lambda only; NOUT = 1 writes lambda per point,
// NOUT = 0 only reduces.
template <class T, int D, int NOUT_>
struct WaveSpeedOp {
    static constexpr int NIN = D + 2;
    static constexpr int NOUT = NOUT_;
    static constexpr bool HAS_LAMBDA = true;
    static constexpr bool ALIASED = false;
    struct State {
        T lam;
    };
    __device__ __forceinline__ static State prepare(const T (&in)[NIN], const Consts<T>& k) {
        const T rho = in[0];
        T m[D];
#pragma unroll
        for (int j = 0; j < D; ++j) m[j] = in[1 + j];
        const T msq = sum_sq<D>(m);
        const T p = pressure(k, rho, msq, in[D + 1]);
        return State{sqrt(msq / (rho * rho)) + sound_speed(k, rho, p)};
    }
    __device__ __forceinline__ static T out(const State& s, int, const Consts<T>&) { return s.lam; }
    __device__ __forceinline__ static T lambda(const State& s, const Consts<T>&) { return s.lam; }
};

// y <- 0.5*sin(x+y): constant(0.5, leaf(y)) * elem_sin(leaf(x) + leaf(y))
// (proj/tests/test_backend.cpp:41).  in = [x, y]; out = [y] (aliased).
template <class T>
struct AxpySinOp {
    static constexpr int NIN = 2;
    static constexpr int NOUT = 1;
    static constexpr bool HAS_LAMBDA = false;
    static constexpr bool ALIASED = true;  // out[0] is in[1]: coherent loads
    struct State {
        T r;
    };
    __device__ __forceinline__ static State prepare(const T (&in)[NIN], const Consts<T>& k) {
        return State{k.half * sin(in[0] + in[1])};
    }
    __device__ __forceinline__ static T out(const State& s, int, const Consts<T>&) { return s.r; }
    __device__ __forceinline__ static T lambda(const State&, const Consts<T>&) { return T(0); }
};

// A contiguous slice [FIRST, FIRST+COUNT) of another Op's outputs, e.g. the
// pressure alone out of cons->prim.  After inlining, state the slice does not
// use is dead and disappears.
template <class Op, int FIRST, int COUNT>
struct SliceOp {
    static constexpr int NIN = Op::NIN;
    static constexpr int NOUT = COUNT;
    static constexpr bool HAS_LAMBDA = false;
    static constexpr bool ALIASED = Op::ALIASED;
    using State = typename Op::State;
    template <class T>
    __device__ __forceinline__ static State prepare(const T (&in)[NIN], const Consts<T>& k) {
        return Op::prepare(in, k);
    }
    template <class T>
    __device__ __forceinline__ static T out(const State& s, int item, const Consts<T>& k) {
        return Op::out(s, FIRST + item, k);
    }
    template <class T>
    __device__ __forceinline__ static T lambda(const State&, const Consts<T>&) {
        return T(0);
    }
};

}  // namespace fvb
