// fft_core.cuh -- register-resident Stockham FFT building blocks for sm_100a.
//
// What is computed (PAPER.md = the paper's LaTeX source):
//   forward  P_k = sum_j p_j w_N^{+jk}, w_N = e^{2 pi i/N}   (eq:DFT)
//   inverse  p_j = sum_k P_k w_N^{-jk}  (the iDFT kernel of PAPER.md:151-153; the
//            1/N is folded into the caller's k-space multiplier)
// The direction is a compile-time flag: the inverse uses the conjugate radix
// kernels and conjugate twiddles, which costs the same instructions as the
// forward (no conjugation passes).
//
// How (not the paper's recursive radix-2 text, which is prior art, but the
// same result): a self-sorting Stockham factorisation N = E^s * r with radix
// E = 16 (built as 4x4) in registers, a final radix r in {2,4,8,16}, and an
// exchange through shared memory between stages.  Thread t of a transform
// holds x[t + TPT*e] (e < E, TPT = N/E threads) on entry and X[t + TPT*e] on
// exit, so global loads and stores are unit-stride across threads.
// Twiddles come from a stage-major table computed on the host in fp64 per
// index (never by recurrence) and rounded once to fp32 for complex64.
#pragma once
#include <type_traits>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fftpde {

template <typename T> struct cplx_t;
template <> struct cplx_t<double> { using type = double2; };
template <> struct cplx_t<float> { using type = float2; };

template <typename C> __device__ __forceinline__ C cadd(C a, C b) { return {a.x + b.x, a.y + b.y}; }
template <typename C> __device__ __forceinline__ C csub(C a, C b) { return {a.x - b.x, a.y - b.y}; }
template <typename C> __device__ __forceinline__ C cconj(C a) { return {a.x, -a.y}; }
template <typename C, typename T> __device__ __forceinline__ C cscale(C a, T s) { return {a.x * s, a.y * s}; }

// a * w (forward) or a * conj(w) (inverse)
template <bool INV, typename C> __device__ __forceinline__ C cmulw(C a, C w)
{
    if constexpr (!INV) return {a.x * w.x - a.y * w.y, a.x * w.y + a.y * w.x};
    else return {a.x * w.x + a.y * w.y, a.y * w.x - a.x * w.y};
}
// a * i^{+1} (forward) or a * i^{-1} (inverse)
template <bool INV, typename C> __device__ __forceinline__ C cmul_i(C a)
{
    if constexpr (!INV) return {-a.y, a.x};
    else return {a.y, -a.x};
}
// a * w_8^{+-1} = a (1 +- i)/sqrt2
template <bool INV, typename C> __device__ __forceinline__ C cmul_w8(C a)
{
    using T = decltype(a.x);
    const T h = (T)0.70710678118654752440084436210485;
    if constexpr (!INV) return {(a.x - a.y) * h, (a.x + a.y) * h};
    else return {(a.x + a.y) * h, (a.y - a.x) * h};
}
// a * w_8^{+-3} = a (-1 +- i)/sqrt2
template <bool INV, typename C> __device__ __forceinline__ C cmul_w83(C a)
{
    using T = decltype(a.x);
    const T h = (T)0.70710678118654752440084436210485;
    if constexpr (!INV) return {-(a.x + a.y) * h, (a.x - a.y) * h};
    else return {(a.y - a.x) * h, -(a.x + a.y) * h};
}

// The Poisson multiplier -scale/|k|^2 (eq:SolutionPoisson; k = 0
// zeroed, R5).  scale = 1/(nx ny) is a power of two, so -scale * rcp_rn(k2) equals
// the IEEE quotient -scale / k2 bit for bit (outside subnormals) while avoiding the
// division's slow path (the C4 column pass spent 5% of its samples in FCHK + MUFU).
__device__ __forceinline__ float poisson_mul(float k2, float scale)
{
    return k2 == 0.f ? 0.f : -scale * __frcp_rn(k2);
}
__device__ __forceinline__ double poisson_mul(double k2, double scale)
{
    return k2 == 0.0 ? 0.0 : -scale * __drcp_rn(k2);
}

// ---------------------------------------------------------------------------
// Small DFTs X_k = sum_n a_n w_R^{+-nk}, in place, natural order in and out.

template <typename C> __device__ __forceinline__ void dft2(C &a0, C &a1)
{
    C t = a0;
    a0 = cadd(t, a1);
    a1 = csub(t, a1);
}

template <bool INV, typename C> __device__ __forceinline__ void dft4(C &a0, C &a1, C &a2, C &a3)
{
    C t0 = cadd(a0, a2), t1 = csub(a0, a2), t2 = cadd(a1, a3), t3 = cmul_i<INV>(csub(a1, a3));
    a0 = cadd(t0, t2);
    a2 = csub(t0, t2);
    a1 = cadd(t1, t3);
    a3 = csub(t1, t3);
}

// radix-8 as 2 x 4: n = 4 n1 + n2, k = k1 + 2 k2, internal twiddle w_8^{n2 k1}
template <bool INV, typename C> __device__ __forceinline__ void dft8(C (&v)[8])
{
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) dft2(v[n2], v[n2 + 4]);   // Y[n2][k1] at v[n2 + 4 k1]
    v[5] = cmul_w8<INV>(v[5]);
    v[6] = cmul_i<INV>(v[6]);
    v[7] = cmul_w83<INV>(v[7]);
    dft4<INV>(v[0], v[1], v[2], v[3]);                     // k1 = 0 -> X[2 k2]     at v[k2]
    dft4<INV>(v[4], v[5], v[6], v[7]);                     // k1 = 1 -> X[1 + 2 k2] at v[4 + k2]
    C o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = v[4 * (k % 2) + k / 2];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = o[k];
}

// radix-16 as 4 x 4: n = 4 n1 + n2, k = k1 + 4 k2, internal twiddle w16^{n2 k1}
template <bool INV, typename C> __device__ __forceinline__ void dft16(C (&v)[16])
{
    using T = decltype(v[0].x);
    const T c1 = (T)0.92387953251128675612818318939679;   // cos(pi/8)
    const T s1 = (T)0.38268343236508977172845998403040;   // sin(pi/8)
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) dft4<INV>(v[n2], v[n2 + 4], v[n2 + 8], v[n2 + 12]);
    // v[n2 + 4 k1] = Y[n2][k1]; multiply by w16^{n2 k1}
    const C w1 = {c1, s1}, w3 = {s1, c1}, w9 = {-c1, -s1};
    v[5] = cmulw<INV>(v[5], w1);     // n2=1,k1=1: w^1
    v[6] = cmul_w8<INV>(v[6]);       // n2=2,k1=1: w^2
    v[7] = cmulw<INV>(v[7], w3);     // n2=3,k1=1: w^3
    v[9] = cmul_w8<INV>(v[9]);       // n2=1,k1=2: w^2
    v[10] = cmul_i<INV>(v[10]);      // n2=2,k1=2: w^4
    v[11] = cmul_w83<INV>(v[11]);    // n2=3,k1=2: w^6
    v[13] = cmulw<INV>(v[13], w3);   // n2=1,k1=3: w^3
    v[14] = cmul_w83<INV>(v[14]);    // n2=2,k1=3: w^6
    v[15] = cmulw<INV>(v[15], w9);   // n2=3,k1=3: w^9
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft4<INV>(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
    C o[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) o[k] = v[4 * (k % 4) + k / 4];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = o[k];
}

// radix-32 as 2 x 16: n = 16 n1 + n2, k = k1 + 2 k2, internal twiddle w32^{n2 k1}
template <bool INV, typename C> __device__ __forceinline__ void dft32(C (&v)[32])
{
    using T = decltype(v[0].x);
    // cos / sin (2 pi j / 32), j = 0..8
    constexpr double cs[9] = {1.0, 0.98078528040323044912618223613424, 0.92387953251128675612818318939679,
                              0.83146961230254523707878837761791, 0.70710678118654752440084436210485,
                              0.55557023301960222474283081394853, 0.38268343236508977172845998403040,
                              0.19509032201612826784828486847702, 0.0};
#pragma unroll
    for (int n2 = 0; n2 < 16; ++n2) dft2(v[n2], v[n2 + 16]);       // Y[n2][k1] at v[n2 + 16 k1]
#pragma unroll
    for (int n2 = 1; n2 < 16; ++n2) {                               // Y[n2][1] *= w32^{n2}
        const T c = (T)(n2 <= 8 ? cs[n2] : -cs[16 - n2]);
        const T s = (T)(n2 <= 8 ? cs[8 - n2] : cs[n2 - 8]);
        v[16 + n2] = cmulw<INV>(v[16 + n2], C{c, s});
    }
    C a[16], b[16];
#pragma unroll
    for (int n2 = 0; n2 < 16; ++n2) { a[n2] = v[n2]; b[n2] = v[16 + n2]; }
    dft16<INV>(a);                                                   // X[2 k2]
    dft16<INV>(b);                                                   // X[1 + 2 k2]
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) { v[2 * k2] = a[k2]; v[2 * k2 + 1] = b[k2]; }
}

template <int R, bool INV, typename C> __device__ __forceinline__ void dft_r(C (&v)[R])
{
    if constexpr (R == 2) dft2(v[0], v[1]);
    else if constexpr (R == 4) dft4<INV>(v[0], v[1], v[2], v[3]);
    else if constexpr (R == 8) dft8<INV>(v);
    else if constexpr (R == 16) dft16<INV>(v);
    else if constexpr (R == 32) dft32<INV>(v);
    else static_assert(R == 1, "radix");
}

// ---------------------------------------------------------------------------
// Compile-time shape of one length-N transform.
template <int N_, int EMAX = 16> struct Shape {
    static constexpr int N = N_;
    static constexpr int E = N_ < EMAX ? N_ : EMAX;    // elements per thread (the radix)
    static constexpr int TPT = N_ / E;                   // threads per transform
    static constexpr int LOGE = E == 32 ? 5 : E == 16 ? 4 : E == 8 ? 3 : E == 4 ? 2 : E == 2 ? 1 : 0;
    // padded smem index: one pad slot every E elements (conflict-free stage-1 scatter)
    static constexpr int PADDED = N_ + (N_ >> LOGE);
    // number of full radix-E stages before the last one, and the last radix
    static constexpr int STAGES = []() { int ns = 1, s = 0; while (ns * E < N_) { ns *= E; ++s; } return s; }();
    static constexpr int NS_LAST = []() { int ns = 1; while (ns * E < N_) ns *= E; return ns; }();
    static constexpr int R_LAST = N_ / NS_LAST;
    // Stage-major twiddle table (built on the host by the same rule): for each
    // middle stage s >= 1 (Ns = E^s) the block tw[m Ns + k] = w_{Ns E}^{m k},
    // m < E, k < Ns; then the last stage tw[m NS_LAST + j] = w_N^{m j}, m < R_LAST.
    // Threads of a warp have consecutive k (or j), so every twiddle load of a
    // warp reads one contiguous run: coalesced, 4 lines per instruction.
    static constexpr int TW_LAST_OFF = []() { int ns = E, off = 0; while (ns * E < N_) { off += E * ns; ns *= E; } return off; }();
    static constexpr int TW_SIZE = NS_LAST > 1 ? TW_LAST_OFF + R_LAST * NS_LAST : 0;
};

// Twiddle load through the read-only path.  volatile: one load per use, so the
// compiler neither keeps a whole table of twiddles live across transforms (CSE)
// nor hoists them far ahead of their use (register pressure).
__device__ __forceinline__ double2 ldtw(const double2 *p)
{
    double2 r;
    asm volatile("ld.global.ca.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ float2 ldtw(const float2 *p)
{
    float2 r;
    asm volatile("ld.global.ca.v2.f32 {%0, %1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p) : "memory");
    return r;
}

// Identity the compiler cannot see through: keeps per-transform index
// arithmetic (twiddle addresses) from being shared across the several
// transforms of one kernel, which would keep ~60 address registers live.
__device__ __forceinline__ int opaque(int x)
{
    int y;
    asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}

template <typename P> __device__ __forceinline__ P *opaque_ptr(P *x)
{
    P *y;
    asm volatile("mov.b64 %0, %1;" : "=l"(y) : "l"(x));
    return y;
}

__device__ __forceinline__ int padidx(int p, int loge) { return p + (p >> loge); }

// Programmatic dependent launch (sm_90+): a pass launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its
// predecessor drains; pdl_wait() blocks until the predecessor grid has completed
// and its memory is visible (a no-op for a normally launched grid), so every pass
// calls it before its first access to a field buffer (constant tables may be read
// before).  pdl_trigger() lets the successor grid launch once every CTA of this
// grid has triggered or exited.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Exchange buffer of one transform: element p lives at base[pad(p) * STRIDE],
// pad(p) = p + p / 2^LOGE (one pad slot every E elements).  For an access
// p0 + d where p0 or d is a multiple of 2^LOGE, pad(p0 + d) = pad(p0) + pad(d),
// so every access of a stage is one base register plus an immediate offset.
template <typename C, int LOGE, int STRIDE> struct SmemView {
    C *base;
    __device__ __forceinline__ C *ptr(int p) const { return base + padidx(p, LOGE) * STRIDE; }
    static __device__ __forceinline__ constexpr int off(int d) { return (d + (d >> LOGE)) * STRIDE; }
    __device__ __forceinline__ C &at(int p) const { return base[padidx(p, LOGE) * STRIDE]; }
};

// Twiddle providers.  mid(s, m) is w_{Ns E}^{m k} of middle stage s >= 1
// (k = t mod Ns), last(q, m) is w_N^{m j} of the last stage (j = t + q TPT),
// both read from the stage-major table of Shape<N>.  TwL1 loads each twiddle
// at its use (L1-resident table); TwReg loads a thread's twiddles once (a
// persistent kernel reuses them for every line it transforms).
template <int N, typename C, int EMAX = 16> struct TwL1 {
    const C *tw;
    int t;
    __device__ __forceinline__ C mid(int s, int m) const
    {
        using S = Shape<N, EMAX>;
        int ns = S::E, off = 0;
#pragma unroll
        for (int i = 1; i < s; ++i) { off += S::E * ns; ns *= S::E; }
        return ldtw(tw + off + opaque(t & (ns - 1)) + m * ns);
    }
    __device__ __forceinline__ C last(int q, int m) const
    {
        using S = Shape<N, EMAX>;
        return ldtw(tw + S::TW_LAST_OFF + opaque(t + q * S::TPT) + m * S::NS_LAST);
    }
};

// As TwL1, but the last stage's twiddles w_N^{m j} (m = 2 .. R-1) are formed
// from the one loaded value w_N^{j} by repeated multiplication (one table load
// per butterfly instead of R-1; a few ulp of extra rounding): for passes whose
// last-stage table reads dominate their L2 -> L1 traffic.
#ifndef FFTPDE_TWPOW
#define FFTPDE_TWPOW 1
#endif
template <int N, typename C, int EMAX = 16> struct TwL1Pow : TwL1<N, C, EMAX> {
    static constexpr bool LAST_POW = true;
};
// TwL1 with radix-32 middle / last stages in the split product form (10 table loads
// per butterfly instead of 31; one extra rounding)
template <int N, typename C, int EMAX = 16> struct TwL1PowSplit : TwL1<N, C, EMAX> {
    static constexpr bool LAST_POW = true, MID_SPLIT = true;
};
template <int N, typename C, int EMAX = 16> struct TwL1Split : TwL1<N, C, EMAX> {
    static constexpr bool LAST_SPLIT = true, MID_SPLIT = true;
};
template <typename Tw, typename = void> struct TwLastPow { static constexpr bool value = false; };
template <typename Tw> struct TwLastPow<Tw, std::void_t<decltype(Tw::LAST_POW)>> { static constexpr bool value = Tw::LAST_POW; };
// LAST_SPLIT (radix-32 last stages): w^{m j}, m = 8 a + b, as the product of the two
// table values w^{8 a j} and w^{b j} (10 loads instead of 31, one extra rounding)
template <typename Tw, typename = void> struct TwLastSplit { static constexpr bool value = false; };
template <typename Tw> struct TwLastSplit<Tw, std::void_t<decltype(Tw::LAST_SPLIT)>> { static constexpr bool value = Tw::LAST_SPLIT; };
// MID_SPLIT (radix-32 middle stages): the same product form for w_{Ns E}^{m k}
template <typename Tw, typename = void> struct TwMidSplit { static constexpr bool value = false; };
template <typename Tw> struct TwMidSplit<Tw, std::void_t<decltype(Tw::MID_SPLIT)>> { static constexpr bool value = Tw::MID_SPLIT; };

// As TwL1, reading a copy of the table staged in shared memory (short kernels
// whose critical path would otherwise wait on L2 twiddle loads every stage).
template <int N, typename C, int EMAX = 16> struct TwSmem {
    const C *tw;
    int t;
    __device__ __forceinline__ C mid(int s, int m) const
    {
        using S = Shape<N, EMAX>;
        int ns = S::E, off = 0;
#pragma unroll
        for (int i = 1; i < s; ++i) { off += S::E * ns; ns *= S::E; }
        return tw[off + (t & (ns - 1)) + m * ns];
    }
    __device__ __forceinline__ C last(int q, int m) const
    {
        using S = Shape<N, EMAX>;
        return tw[S::TW_LAST_OFF + t + q * S::TPT + m * S::NS_LAST];
    }
};

// As TwSmem for complex128, each read a volatile ld.shared at its use (like ldtw:
// neither kept live across transforms nor hoisted), `base` the table's shared-window
// address.
template <int N, int EMAX = 16> struct TwSmemV {
    uint32_t base;
    int t;
    static __device__ __forceinline__ double2 ld(uint32_t a)
    {
        double2 r;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "r"(a));
        return r;
    }
    __device__ __forceinline__ double2 mid(int s, int m) const
    {
        using S = Shape<N, EMAX>;
        int ns = S::E, off = 0;
#pragma unroll
        for (int i = 1; i < s; ++i) { off += S::E * ns; ns *= S::E; }
        return ld(base + 16u * (uint32_t)(off + (t & (ns - 1)) + m * ns));
    }
    __device__ __forceinline__ double2 last(int q, int m) const
    {
        using S = Shape<N, EMAX>;
        return ld(base + 16u * (uint32_t)(S::TW_LAST_OFF + t + q * S::TPT + m * S::NS_LAST));
    }
};

template <int N, int EMAX = 16> struct TwSmemVSplit : TwSmemV<N, EMAX> {
    static constexpr bool LAST_SPLIT = true;
};

template <int N, typename C, int EMAX = 16> struct TwReg {
    using S = Shape<N, EMAX>;
    static constexpr int NMID = S::STAGES > 1 ? (S::STAGES - 1) * (S::E - 1) : 1;
    static constexpr int Q = S::E / S::R_LAST;
    static constexpr int NLAST = S::R_LAST > 1 ? Q * (S::R_LAST - 1) : 1;
    C wm[NMID];
    C wl[NLAST];
    __device__ __forceinline__ void load(const C *tw, int t)
    {
        TwL1<N, C, EMAX> l{tw, t};
#pragma unroll
        for (int s = 1; s < S::STAGES; ++s)
#pragma unroll
            for (int m = 1; m < S::E; ++m) wm[(s - 1) * (S::E - 1) + m - 1] = l.mid(s, m);
        if (S::NS_LAST > 1) {
#pragma unroll
            for (int q = 0; q < Q; ++q)
#pragma unroll
                for (int m = 1; m < S::R_LAST; ++m) wl[q * (S::R_LAST - 1) + m - 1] = l.last(q, m);
        }
    }
    __device__ __forceinline__ C mid(int s, int m) const { return wm[(s - 1) * (S::E - 1) + m - 1]; }
    __device__ __forceinline__ C last(int q, int m) const { return wl[q * (S::R_LAST - 1) + m - 1]; }
};

// Transform of one length-N sequence held as v[e] = x[t + TPT e]; on exit
// v[e] = X[t + TPT e].  INV selects the conjugate kernel (inverse direction,
// unscaled).  `sync` synchronises the threads sharing the exchange buffer
// (warp, line or CTA); the buffer is free again when this returns.
#ifndef FFTPDE_TG32
#define FFTPDE_TG32 8      // twiddles loaded per group by the radix-32 stages
#endif
template <int N, bool INV, int EMAX = 16, typename C, typename View, typename Tw, typename Sync>
__device__ __forceinline__ void fft_tw(C (&v)[Shape<N, EMAX>::E], const View &sm, int t, const Tw &tw,
                                       Sync sync)
{
    using S = Shape<N, EMAX>;
    constexpr int E = S::E, TPT = S::TPT;
    // Twiddles fetched from memory (TwL1) are loaded in groups of TG before their
    // multiplies, so a group's loads are in flight together instead of each load's
    // latency following the previous multiply (the loads are volatile and ordered).
    constexpr int TG = E <= 1 ? 1 : E <= 16 ? E - 1 : FFTPDE_TG32;
    int Ns = 1;
#pragma unroll
    for (int s = 0; s < S::STAGES; ++s) {
        const int k = t & (Ns - 1);
        if (s > 0 && E == 32 && TwMidSplit<Tw>::value) {
            C wb[8], wa[4];
#pragma unroll
            for (int b = 1; b < 8; ++b) wb[b] = tw.mid(s, b);
#pragma unroll
            for (int a = 1; a < 4; ++a) wa[a] = tw.mid(s, 8 * a);
#pragma unroll
            for (int m = 1; m < E; ++m) {
                const int a = m / 8, b = m % 8;
                C w;
                if (a == 0) w = wb[b];
                else if (b == 0) w = wa[a];
                else w = C{wa[a].x * wb[b].x - wa[a].y * wb[b].y, wa[a].x * wb[b].y + wa[a].y * wb[b].x};
                v[m] = cmulw<INV>(v[m], w);
            }
        } else if (s > 0) {
#pragma unroll
            for (int m0 = 1; m0 < E; m0 += TG) {
                C w[TG];
#pragma unroll
                for (int j = 0; j < TG; ++j)
                    if (m0 + j < E) w[j] = tw.mid(s, m0 + j);
#pragma unroll
                for (int j = 0; j < TG; ++j)
                    if (m0 + j < E) v[m0 + j] = cmulw<INV>(v[m0 + j], w[j]);
            }
        }
        dft_r<E, INV>(v);
        // scatter X_m of butterfly t to (t / Ns) Ns E + k + m Ns; base or m Ns is a multiple of E
        C *wp = sm.ptr((t - k) * E + k);
#pragma unroll
        for (int m = 0; m < E; ++m) wp[View::off(m * Ns)] = v[m];
        sync();
        if constexpr (TPT % E == 0) {
            const C *rp = sm.ptr(t);
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = rp[View::off(m * TPT)];
        } else {
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = sm.at(t + m * TPT);
        }
        sync();
        Ns *= E;
    }
    // last stage: radix R = N / Ns, E/R butterflies per thread, j = t + q TPT,
    // inputs x[j + m N/R] = slot q + m E/R, outputs X[j + m Ns] -> same slots.
    constexpr int R = S::R_LAST;
    constexpr int Q = E / R;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        C u[R];
#pragma unroll
        for (int m = 0; m < R; ++m) u[m] = v[q + m * Q];
        if constexpr (S::NS_LAST > 1 && R == 32 && TwLastSplit<Tw>::value) {
            C wb[8], wa[4];
#pragma unroll
            for (int b = 1; b < 8; ++b) wb[b] = tw.last(q, b);
#pragma unroll
            for (int a = 1; a < 4; ++a) wa[a] = tw.last(q, 8 * a);
#pragma unroll
            for (int m = 1; m < R; ++m) {
                const int a = m / 8, b = m % 8;
                C w;
                if (a == 0) w = wb[b];
                else if (b == 0) w = wa[a];
                else w = C{wa[a].x * wb[b].x - wa[a].y * wb[b].y, wa[a].x * wb[b].y + wa[a].y * wb[b].x};
                u[m] = cmulw<INV>(u[m], w);
            }
        } else if constexpr (S::NS_LAST > 1 && TwLastPow<Tw>::value) {
            const C w1 = tw.last(q, 1);
            C wm = w1;
#pragma unroll
            for (int m = 1; m < R; ++m) {
                if (m > 1) wm = C{wm.x * w1.x - wm.y * w1.y, wm.x * w1.y + wm.y * w1.x};
                u[m] = cmulw<INV>(u[m], wm);
            }
        } else if (S::NS_LAST > 1) {
            constexpr int LG = R <= 1 ? 1 : R <= 16 ? R - 1 : 8;
#pragma unroll
            for (int m0 = 1; m0 < R; m0 += LG) {
                C w[LG];
#pragma unroll
                for (int j = 0; j < LG; ++j)
                    if (m0 + j < R) w[j] = tw.last(q, m0 + j);
#pragma unroll
                for (int j = 0; j < LG; ++j)
                    if (m0 + j < R) u[m0 + j] = cmulw<INV>(u[m0 + j], w[j]);
            }
        }
        dft_r<R, INV>(u);
#pragma unroll
        for (int m = 0; m < R; ++m) v[q + m * Q] = u[m];
    }
}

// Twiddles loaded from the table at each use.
template <int N, bool INV, int EMAX = 16, typename C, typename View, typename Sync>
__device__ __forceinline__ void fft(C (&v)[Shape<N, EMAX>::E], const View &sm, int t,
                                    const C *__restrict__ tw, Sync sync)
{
#if FFTPDE_TWPOW
    // last radix 4 or 8: one table load per butterfly, powers by multiplication
    // (C5 row and column passes -1%, C3 wave pass -5%; FFTPDE_TWPOW=0 restores the loads)
    if constexpr (Shape<N, EMAX>::R_LAST <= 8 && Shape<N, EMAX>::R_LAST > 2)
        fft_tw<N, INV, EMAX>(v, sm, t, TwL1Pow<N, C, EMAX>{{tw, t}}, sync);
    else
#endif
    fft_tw<N, INV, EMAX>(v, sm, t, TwL1<N, C, EMAX>{tw, t}, sync);
}

struct SyncCTA { __device__ __forceinline__ void operator()() const { __syncthreads(); } };
struct SyncWarp { __device__ __forceinline__ void operator()() const { __syncwarp(); } };

} // namespace fftpde
