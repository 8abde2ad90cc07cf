// rr_march.cuh — device code of the march kernels (included by the
// rr_k_*.cu translation units, each instantiating one metric family so the
// build runs in parallel).  See the file comment below for the reference map.
#pragma once
// rr_kernels.cu — sm_100a kernels of the B200 geodesic tracer.
//
// K1 raygen (fused prologue)  <- pixel_direction   src/render/camera.cpp:22-29
// K2 march                    <- march_group       include/rray/render/detail/kernel_impl.hpp:22-94
//                                + flow_step_t     include/rray/geodesics/integrate.hpp:46-99
//                                + christoffel_eval include/rray/metrics/metric.hpp:69-105
//                                + intersect_segment src/render/scene.cpp:15-109
// K3 shade (fused epilogue)   <- shade             src/render/render.cpp:14-25
// K6 detile                   <- (none: the reference is single-process)
// See rr_device.cuh for the math and DESIGN.md for the roofline.
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "rr_device.cuh"
#include "rr_internal.h"

namespace rr {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kThreads = 128;   // 4 warps per CTA
#ifndef RR_FAST_SINCOS
#define RR_FAST_SINCOS 1
#endif
#ifndef RR_GROUP_TESTS
#define RR_GROUP_TESTS 1
#endif
#ifndef RR_RAY_PAIRS
// 1: Gaussian-bump frames march two rays per thread with packed FP32
// (march2_kernel); 0: one ray per thread (march_kernel) for every scene.
#define RR_RAY_PAIRS 1
#endif
#ifndef RR_TWIST_PAIRS
// 1: single-twist RK4 frames (C4, meshes included) on the ray-pair kernel
#define RR_TWIST_PAIRS 1
#endif
#ifndef RR_TWIST_PAIRS_MESH
// 1: single-twist RK4 frames WITH meshes on the ray-pair kernel too
#define RR_TWIST_PAIRS_MESH 0
#endif
#ifndef RR_RK23_PAIRS
// 1: Gaussian-bump rk23 frames (mesh-free) on the ray-pair kernel
#define RR_RK23_PAIRS 1
#endif
#ifndef RR_RK23_K1_PRELOOP
// 1: the rk23 ray-pair march evaluates every ray's first k1 before its loop
#define RR_RK23_K1_PRELOOP 1
#endif
#ifndef RR_X2_SCALAR_CONSTS_LIT
// bump constants as scalars (DevBumpS: UR.F32 broadcast operands, 5 instead of
// 10 LDCU.64 per bump) in rk23 (and, with 1 here, in the lit marches: they won
// inside the single fused lit launch, 15.55 -> 15.47 ms, but the two separate
// lit launches run 0.25% faster on the broadcast pairs (DevBumpB) that the
// unlit frames use: profiles/r2z_scalar_consts_ab.log, r2z_litvec_ab.log)
#define RR_X2_SCALAR_CONSTS_LIT 0
#endif
#ifndef RR_X2_SCALAR_CONSTS_RK23
#define RR_X2_SCALAR_CONSTS_RK23 1
#endif
#ifndef RR_TWIST_ONE_STATIC
// 1: the one-ray kernel for single-twist scenes with meshes is a variant
// without the general diffeo fold (rr_k_diffeo.cu)
#define RR_TWIST_ONE_STATIC 1
#endif
#ifndef RR_EUCLID_PREFETCH
#define RR_EUCLID_PREFETCH 1   // one-ray Euclidean launches fetch their next unit index one unit ahead
#endif
#ifndef RR_BOUNDS_BUDGET
// 1: the single-twist ray-pair march tests a chord end against the bounds box
// only once the chords since the last test have used up that point's distance
// to the box
#define RR_BOUNDS_BUDGET 1
#endif
#ifndef RR_SMALL_LAUNCH_CTAS
#define RR_SMALL_LAUNCH_CTAS 1   // ray-pair launches with few items per SM use fewer CTAs per SM
#endif
#ifndef RR_CHAIN_STATIC
// 1: two-stage twist/bend chains use a fold specialised at compile time
// (rr_k_pair_chain.cu); others (and 0) the run-time stage loop
#define RR_CHAIN_STATIC 1
#endif
#ifndef RR_X2_HITS_STAGED
// 1: primary hit records of the lit launch are produced after the unit's
// march from shared-memory staged chords (hit_normal out of the march loop)
#define RR_X2_HITS_STAGED 1
#endif
#ifndef RR_COUNT_OWN_MASK
#define RR_COUNT_OWN_MASK 0   // diagnostics build: count each ray's own culling mask, not the warp union
#endif
#ifndef RR_CHAIN_PAIRS
// 1: general diffeo chains (RK4) on the ray-pair kernel (kDiffeoChain)
#define RR_CHAIN_PAIRS 1
#endif
#ifndef RR_CHAIN_PAIRS_MESH
#define RR_CHAIN_PAIRS_MESH 1
#endif
#ifndef RR_X2_KAHAN
// compensated position sums in the ray-pair march.  Without them C3 runs 1.3%
// faster but C1 (2000-step marches at h = 0.01) reaches 7.4e-5 endpoint error
// against the 1e-4 contract (3.2e-5 with them): profiles/r2v_kahan_ab.log
#define RR_X2_KAHAN 1
#endif
#ifndef RR_X2_FUSED
// ray-pair frames with lights: 1 = one launch (primary units, then
// (unit, light) shadow units, ready flags); 0 = a hit-record launch + a shadow
// launch, each with its own register budget and half the code.  0 since the
// final round-2 build: 15.32-15.34 ms (shadow launch at 7 CTAs/SM) vs 15.47-
// 15.49 fused, bit-identical (profiles/r2z_unfused_ab.log); in round 1 the
// fused launch had won
#define RR_X2_FUSED 0
#endif
#ifndef RR_X2_RK4_UNROLL
#define RR_X2_RK4_UNROLL 1   // 4 RK4 stages unrolled (4 small bump loops): C3 10.32 -> 9.91 ms, lights 16.94 -> 16.66
#endif
#ifndef RR_X2_BODY
#define RR_X2_BODY 3   // bump body of the ray-pair march: 1 = G accumulated, 3 = T-trick (accel_bumps_x2)
#endif
#ifndef RR_X2_RK4_UNROLL_LIT
#define RR_X2_RK4_UNROLL_LIT RR_X2_RK4_UNROLL
#endif
#ifndef RR_X2_RK4_UNROLL_SHADOW
#define RR_X2_RK4_UNROLL_SHADOW RR_X2_RK4_UNROLL_LIT
#endif
#ifndef RR_MIN_BLOCKS_X2
// ray-pair kernel occupancy (CUDA-event A/B).  Round 1: 6 CTAs (80
// registers) beat 7 on the unlit frame, 9.39 vs 9.63 ms
// (profiles/r1i_shadow_frame.md).  Final round-2 build: 7 (72 registers) ties
// 6 on C3 (9.16 vs 9.15 ms median, 9.09-9.11 vs 9.13-9.15 min) and wins on
// C5 4K (34.98 vs 35.27 ms); the lit hit-record launch keeps 6
// (profiles/r2z_c3occ_ab.log).  The 4-slot variant (C1) uses its own.
#define RR_MIN_BLOCKS_X2 7
#endif
#ifndef RR_MIN_BLOCKS_X2_FUSED
#define RR_MIN_BLOCKS_X2_FUSED 7
#endif
#ifndef RR_MIN_BLOCKS_X2_SMALL
#define RR_MIN_BLOCKS_X2_SMALL 6
#endif
#ifndef RR_MIN_BLOCKS_X2_TWIST
// ray-pair single-twist frames (C4 without meshes): 7 CTAs/SM (72 registers)
// since the bounds budget: 6.24-6.26 vs 6.47-6.50 ms at 6, 7.12 at 8, 7.22 at
// 5 (profiles/r2z_occ_small_twist_ab.log)
#define RR_MIN_BLOCKS_X2_TWIST 7
#endif
#ifndef RR_MIN_BLOCKS_X2_TWIST_MESH
#define RR_MIN_BLOCKS_X2_TWIST_MESH 6   // ray-pair single-twist frames with meshes (C4)
#endif
#ifndef RR_MIN_BLOCKS_X2_CHAIN
// ray-pair general diffeo chains: the packed fold (J, q, w pairs) is register
// heavy; 4 CTAs (128 registers) beat 5 and 6 (twist o bend: 45.1 / 45.9 /
// 48.1 ms, one ray per thread 46.9; with the 100k mesh 46.8 / 47.4 / 49.1 vs
// 49.0; profiles/r2p_chain_ab.log)
#define RR_MIN_BLOCKS_X2_CHAIN 4
#endif
#ifndef RR_MIN_BLOCKS_X2_CHAIN_STATIC
// compile-time chain folds (112-116 registers at 4): 5 CTAs/SM, 96
// registers (C4 twist + bend + mesh 34.0 / 32.7 / 35.7 ms at 4 / 5 / 6,
// profiles/r2z_chain_occupancy_ab.log)
#define RR_MIN_BLOCKS_X2_CHAIN_STATIC 5
#endif
#ifndef RR_MIN_BLOCKS_X2_SHADOW
#define RR_MIN_BLOCKS_X2_SHADOW 7   // the shadow launch of lit frames (72 registers): 15.33 vs 15.37 ms at 6
#endif
#ifndef RR_MIN_BLOCKS_X2_HITS
#define RR_MIN_BLOCKS_X2_HITS 6     // the hit-record launch of lit frames (80 registers)
#endif
#ifndef RR_MIN_BLOCKS_X2_RK23
// ray-pair rk23 (FSAL stage + error terms per ray pair): 7 CTAs/SM (72
// registers) since the pre-loop k1 and scalar constants shrank it: 10.43 /
// 10.48 / 12.97 ms at 6 / 5 / 4 (profiles/r2z_occ_recheck_ab.log), 10.40-10.42
// vs 10.45 at 7 vs 6 (r2z_rk23occ7_ab.log)
#define RR_MIN_BLOCKS_X2_RK23 7
#endif
#ifndef RR_MIN_BLOCKS_RK23
#define RR_MIN_BLOCKS_RK23 5   // rk23 carries the FSAL stage + error terms: <= 96 registers
#endif
#ifndef RR_MIN_BLOCKS
#define RR_MIN_BLOCKS 7   // <= 72 registers: 7 CTAs = 28 warps per SM (measured best)
#endif
#ifndef RR_MIN_BLOCKS_MESH
// mesh variants (BVH stack + free-distance ball): 6 CTAs, C4 twist + mesh
// 12.85 vs 13.2-13.4 ms at 7, 13.1-13.2 at 5, 14.4-14.7 at 8; bend neutral
// (profiles/r1k_minblocks_ab.log); the mesh-free twist stays at 7 (8.09 vs
// 8.32 ms at 6, profiles/r1l_minblocks_nomesh_ab.log)
#define RR_MIN_BLOCKS_MESH 6
#endif

// Device-side bounds / protocol checks (compute-sanitizer is not available
// on this pool): build with -DRR_CHECKS=1 (tools/build_variants.sh) and run
// tools/sanitize_frames.py; a failed check prints its site and traps.
#ifndef RR_CHECKS
#define RR_CHECKS 0
#endif
#if RR_CHECKS
#include <cstdio>
#define RR_CHECK(cond, what)                                                                   \
    do {                                                                                       \
        if (!(cond)) {                                                                         \
            printf("RR_CHECK failed: %s (line %d) block %d thread %d\n", what, __LINE__,     \
                   (int)blockIdx.x, (int)threadIdx.x);                                        \
            __trap();                                                                          \
        }                                                                                      \
    } while (0)
#else
#define RR_CHECK(cond, what) \
    do {                     \
    } while (0)
#endif

struct F3 {
    float x, y, z;
};

__device__ __forceinline__ F3 f3(float x, float y, float z) { return F3{x, y, z}; }

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// ---------------------------------------------------------------------------
// Graph metric, Gaussian bumps only (factored form, rr_device.cuh header).
// `um` is warp-uniform: bit j set <=> bump slot j is evaluated by the whole
// warp this step.  Slot tests cost 2 issue slots each, so NB is the smallest
// of 4/8/16/32 holding the field (a sign-split slot layout was measured
// slower: it doubles the slots tested per evaluation).
template <int NB>
__device__ __forceinline__ F3 accel_bumps(const DevParams& P, uint32_t um, F3 p, F3 y) {
    float Gx = 0.f, Gy = 0.f, Gz = 0.f, Q1 = 0.f, Sx = 0.f, Sy = 0.f, Sz = 0.f;
#pragma unroll
    for (int g = 0; g < NB; g += 4) {
#if RR_GROUP_TESTS
        // slots are sorted by centre x on the host, so a ray's active bumps
        // cluster and whole groups of 4 are skipped with one test
        if (!((um >> g) & 0xFu)) continue;
#endif
#pragma unroll
        for (int j = g; j < g + 4; ++j) {
            if (um & (1u << j)) {
                const DevBump& b = P.bumps[j];
                const float dx = p.x - b.cx, dy = p.y - b.cy, dz = p.z - b.cz;
                const float gx = dx * b.kx, gy = dy * b.ky, gz = dz * b.kz;
                const float q = fmaf(dx, gx, fmaf(dy, gy, fmaf(dz, gz, b.la)));
                const float v = ex2(q) * b.sgn;
                Gx = fmaf(v, gx, Gx);
                Gy = fmaf(v, gy, Gy);
                Gz = fmaf(v, gz, Gz);
                const float t = fmaf(y.x, gx, fmaf(y.y, gy, y.z * gz));
                Q1 = fmaf(v * t, t, Q1);
                Sx = fmaf(v, b.kx, Sx);
                Sy = fmaf(v, b.ky, Sy);
                Sz = fmaf(v, b.kz, Sz);
            }
        }
    }
    // G = beta G';  Q = beta^2 Q1 - beta (Y . S');  a = (Q / (1 + |G|^2)) G
    const float ys = fmaf(y.x * y.x, Sx, fmaf(y.y * y.y, Sy, y.z * y.z * Sz));
    const float Q = fmaf(kBeta * kBeta, Q1, -kBeta * ys);
    const float w = fmaf(kBeta * kBeta, fmaf(Gx, Gx, fmaf(Gy, Gy, Gz * Gz)), 1.f);
    const float r = Q * rcp_approx(w) * kBeta;
    return f3(r * Gx, r * Gy, r * Gz);
}

// ---------------------------------------------------------------------------
// Ray pairs (packed FP32: FADD2 / FMUL2 / FFMA2).  The march is bound by
// issue slots; a thread that carries TWO rays evaluates every per-ray
// operation of both with one packed instruction, with the per-bump constants
// as broadcast 64-bit uniform operands (DevBumpB).  Measured on the bump body
// alone (tools/microbench/bump_body.cu, profiles/r1g_raypair.md): 0.88 vs
// 1.10-1.15 ps per ray-bump at 8 active bumps.  (Pairing two bump SLOTS of one
// ray instead was measured slower: profiles/r1e_ffma2.md.)
typedef unsigned long long u64;
struct F2 {           // (ray 0, ray 1)
    u64 v;
};
__device__ __forceinline__ F2 mk2(float a, float b) {
    F2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ F2 bc2(float a) { return mk2(a, a); }
__device__ __forceinline__ float lo2(F2 x) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x.v));
    return a;
}
__device__ __forceinline__ float hi2(F2 x) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x.v));
    return b;
}
__device__ __forceinline__ float get2(F2 x, int r) { return r ? hi2(x) : lo2(x); }
__device__ __forceinline__ F2 add2(F2 a, F2 b) {
    F2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
__device__ __forceinline__ F2 sub2(F2 a, F2 b) {
    F2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
__device__ __forceinline__ F2 mul2(F2 a, F2 b) {
    F2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
__device__ __forceinline__ F2 fma2(F2 a, F2 b, F2 c) {
    F2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
    return r;
}
// c - a*b as ONE FFMA2 with a negated operand (ptxas folds the pair; f32x2
// has no neg in PTX, and an xor would cost two ALU ops)
__device__ __forceinline__ F2 fnma2(F2 a, F2 b, F2 c) {
    F2 r;
    asm("{\n\t.reg .b64 t;\n\tmul.rn.f32x2 t, %1, %2;\n\tsub.rn.f32x2 %0, %3, t;\n\t}"
        : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
    return r;
}
__device__ __forceinline__ F2 ld2(const float2& f) { return F2{*reinterpret_cast<const u64*>(&f)}; }
// select per ray: r0 ? a.lo : b.lo, r1 ? a.hi : b.hi
__device__ __forceinline__ F2 sel2(bool r0, bool r1, F2 a, F2 b) {
    return mk2(r0 ? lo2(a) : lo2(b), r1 ? hi2(a) : hi2(b));
}

struct P3 {           // a 3-vector for a ray pair
    F2 x, y, z;
};
__device__ __forceinline__ F3 ray_of(const P3& v, int r) { return f3(get2(v.x, r), get2(v.y, r), get2(v.z, r)); }
__device__ __forceinline__ P3 pair_of(F3 a, F3 b) { return P3{mk2(a.x, b.x), mk2(a.y, b.y), mk2(a.z, b.z)}; }

// accel_bumps for a ray pair (same factored form) over the warp-uniform mask
// of the 64 rays: a uniform-datapath loop over the active slots, positive
// amplitudes first, then negative ones with the sign folded into the
// accumulating FFMA2s (negated operand).  Measured alternatives (unrolled
// slot tests, pairs/groups of slots per test, the sign as an XOR, G = p.S - T,
// compact or shared-memory slots): profiles/r1g_raypair.md, r1i_shadow_frame.md.
template <int NB, bool SC = false>
__device__ __forceinline__ P3 accel_bumps_x2(const DevParams& P, uint32_t um, const P3& p, const P3& y) {
    F2 Gx = bc2(0.f), Gy = bc2(0.f), Gz = bc2(0.f), Q1 = bc2(0.f);
    F2 Sx = bc2(0.f), Sy = bc2(0.f), Sz = bc2(0.f);
    auto body = [&](const DevBumpB& b, bool neg) {
        const F2 dx = add2(p.x, ld2(b.ncx)), dy = add2(p.y, ld2(b.ncy)), dz = add2(p.z, ld2(b.ncz));
        const F2 gx = mul2(dx, ld2(b.kx)), gy = mul2(dy, ld2(b.ky)), gz = mul2(dz, ld2(b.kz));
        const F2 q = fma2(dx, gx, fma2(dy, gy, fma2(dz, gz, ld2(b.la))));
        const F2 e = mk2(ex2(lo2(q)), ex2(hi2(q)));
        const F2 t = fma2(y.x, gx, fma2(y.y, gy, mul2(y.z, gz)));
        const F2 et = mul2(e, t);
#if RR_X2_BODY == 3
        // T-trick: accumulate T = sum e K.c (a constant operand: FFMA2 with
        // two register pairs, full rate) instead of G = sum e g (three
        // register pairs, 2/3 rate, tools/microbench/fp32_pipes.cu); G = p.S - T
        // after the loop.  C3 9.45 -> 9.36 ms, full-frame endpoint max
        // 3.04e-5 -> 2.76e-5 (profiles/r2j_body_ab.log)
        const F2 gxx = ld2(b.kcx), gyy = ld2(b.kcy), gzz = ld2(b.kcz);
#else
        const F2 gxx = gx, gyy = gy, gzz = gz;
#endif
        if (neg) {
            Gx = fnma2(e, gxx, Gx);
            Gy = fnma2(e, gyy, Gy);
            Gz = fnma2(e, gzz, Gz);
            Q1 = fnma2(et, t, Q1);
            Sx = fnma2(e, ld2(b.kx), Sx);
            Sy = fnma2(e, ld2(b.ky), Sy);
            Sz = fnma2(e, ld2(b.kz), Sz);
        } else {
            Gx = fma2(e, gxx, Gx);
            Gy = fma2(e, gyy, Gy);
            Gz = fma2(e, gzz, Gz);
            Q1 = fma2(et, t, Q1);
            Sx = fma2(e, ld2(b.kx), Sx);
            Sy = fma2(e, ld2(b.ky), Sy);
            Sz = fma2(e, ld2(b.kz), Sz);
        }
    };
    // SC: the same body over scalar constants: bc2(c) of a uniform scalar is a
    // broadcast UR.F32 operand, and each 64-bit uniform load carries two
    auto body_s = [&](const DevBumpS& b, bool neg) {
        const float2 w0 = b.ncxy, w1 = b.nczkx, w2 = b.kyz, w3 = b.lakcx, w4 = b.kcyz;
        const F2 dx = add2(p.x, bc2(w0.x)), dy = add2(p.y, bc2(w0.y)), dz = add2(p.z, bc2(w1.x));
        const F2 kx = bc2(w1.y), ky = bc2(w2.x), kz = bc2(w2.y);
        const F2 gx = mul2(dx, kx), gy = mul2(dy, ky), gz = mul2(dz, kz);
        const F2 q = fma2(dx, gx, fma2(dy, gy, fma2(dz, gz, bc2(w3.x))));
        const F2 e = mk2(ex2(lo2(q)), ex2(hi2(q)));
        const F2 t = fma2(y.x, gx, fma2(y.y, gy, mul2(y.z, gz)));
        const F2 et = mul2(e, t);
        const F2 gxx = bc2(w3.y), gyy = bc2(w4.x), gzz = bc2(w4.y);   // T-trick (RR_X2_BODY 3)
        if (neg) {
            Gx = fnma2(e, gxx, Gx);
            Gy = fnma2(e, gyy, Gy);
            Gz = fnma2(e, gzz, Gz);
            Q1 = fnma2(et, t, Q1);
            Sx = fnma2(e, kx, Sx);
            Sy = fnma2(e, ky, Sy);
            Sz = fnma2(e, kz, Sz);
        } else {
            Gx = fma2(e, gxx, Gx);
            Gy = fma2(e, gyy, Gy);
            Gz = fma2(e, gzz, Gz);
            Q1 = fma2(et, t, Q1);
            Sx = fma2(e, kx, Sx);
            Sy = fma2(e, ky, Sy);
            Sz = fma2(e, kz, Sz);
        }
    };
    static_assert(!SC || RR_X2_BODY == 3, "scalar constants: T-trick body only");
    uint32_t m = um & ~P.neg_mask;
#pragma unroll 1
    while (m) {
        const int j = __ffs(m) - 1;
        m &= m - 1u;
        if constexpr (SC) body_s(P.bumpss[j], false);
        else body(P.bumpsb[j], false);
    }
    m = um & P.neg_mask;
#pragma unroll 1
    while (m) {
        const int j = __ffs(m) - 1;
        m &= m - 1u;
        if constexpr (SC) body_s(P.bumpss[j], true);
        else body(P.bumpsb[j], true);
    }
#if RR_X2_BODY == 3
    Gx = sub2(mul2(p.x, Sx), Gx);
    Gy = sub2(mul2(p.y, Sy), Gy);
    Gz = sub2(mul2(p.z, Sz), Gz);
#endif
    const F2 ys = fma2(mul2(y.x, y.x), Sx, fma2(mul2(y.y, y.y), Sy, mul2(mul2(y.z, y.z), Sz)));
    const F2 Q = fma2(bc2(kBeta * kBeta), Q1, mul2(bc2(-kBeta), ys));
    const F2 w = fma2(bc2(kBeta * kBeta), fma2(Gx, Gx, fma2(Gy, Gy, mul2(Gz, Gz))), bc2(1.f));
    const F2 r = mul2(mul2(Q, mk2(rcp_approx(lo2(w)), rcp_approx(hi2(w)))), bc2(kBeta));
    return P3{mul2(r, Gx), mul2(r, Gy), mul2(r, Gz)};
}

// ---------------------------------------------------------------------------
// Graph metric, general field: any number of bumps (<= kMaxBumps) plus
// polynomial terms (scalar_field.hpp:128-161); full gradient + Hessian.
__device__ __forceinline__ F3 accel_graph_general(const DevParams& P, F3 p, F3 y) {
    float fx = 0.f, fy = 0.f, fz = 0.f;                               // grad f
    float hxx = 0.f, hxy = 0.f, hxz = 0.f, hyy = 0.f, hyz = 0.f, hzz = 0.f;
    for (int j = 0; j < P.n_bumps; ++j) {
        const DevBump& b = P.bumps[j];
        const float dx = p.x - b.cx, dy = p.y - b.cy, dz = p.z - b.cz;
        const float gx = dx * b.kx * kBeta, gy = dy * b.ky * kBeta, gz = dz * b.kz * kBeta;
        const float v = ex2(fmaf(dx * b.kx, dx, fmaf(dy * b.ky, dy, fmaf(dz * b.kz, dz, b.la)))) * b.sgn;
        fx = fmaf(-v, gx, fx);
        fy = fmaf(-v, gy, fy);
        fz = fmaf(-v, gz, fz);
        hxx = fmaf(v, fmaf(gx, gx, -b.kx * kBeta), hxx);
        hyy = fmaf(v, fmaf(gy, gy, -b.ky * kBeta), hyy);
        hzz = fmaf(v, fmaf(gz, gz, -b.kz * kBeta), hzz);
        hxy = fmaf(v, gx * gy, hxy);
        hxz = fmaf(v, gx * gz, hxz);
        hyz = fmaf(v, gy * gz, hyz);
    }
    if (P.n_poly > 0) {
        float xp[5], yp[5], zp[5];
        xp[0] = yp[0] = zp[0] = 1.f;
#pragma unroll
        for (int k = 1; k < 5; ++k) {
            xp[k] = xp[k - 1] * p.x;
            yp[k] = yp[k - 1] * p.y;
            zp[k] = zp[k - 1] * p.z;
        }
        for (int i = 0; i < P.n_poly; ++i) {
            const DevPoly& t = P.poly[i];
            const int a = t.a, b = t.b, c = t.c;
            const float xa = xp[a], yb = yp[b], zc = zp[c];
            const float xa1 = a > 0 ? xp[a - 1] : 0.f, yb1 = b > 0 ? yp[b - 1] : 0.f;
            const float zc1 = c > 0 ? zp[c - 1] : 0.f;
            const float xa2 = a > 1 ? xp[a - 2] : 0.f, yb2 = b > 1 ? yp[b - 2] : 0.f;
            const float zc2 = c > 1 ? zp[c - 2] : 0.f;
            fx = fmaf(t.coef * a, xa1 * yb * zc, fx);
            fy = fmaf(t.coef * b, xa * yb1 * zc, fy);
            fz = fmaf(t.coef * c, xa * yb * zc1, fz);
            hxx = fmaf(t.coef * (a * (a - 1)), xa2 * yb * zc, hxx);
            hyy = fmaf(t.coef * (b * (b - 1)), xa * yb2 * zc, hyy);
            hzz = fmaf(t.coef * (c * (c - 1)), xa * yb * zc2, hzz);
            hxy = fmaf(t.coef * (a * b), xa1 * yb1 * zc, hxy);
            hxz = fmaf(t.coef * (a * c), xa1 * yb * zc1, hxz);
            hyz = fmaf(t.coef * (b * c), xa * yb1 * zc1, hyz);
        }
    }
    // Q = y^T H y;  a = -(Q / (1 + |grad f|^2)) grad f   (metric.hpp:74-83)
    const float Q = hxx * y.x * y.x + hyy * y.y * y.y + hzz * y.z * y.z +
                    2.f * (hxy * y.x * y.y + hxz * y.x * y.z + hyz * y.y * y.z);
    const float w = 1.f + fx * fx + fy * fy + fz * fz;
    const float r = -Q * rcp_approx(w);
    return f3(r * fx, r * fy, r * fz);
}

// ---------------------------------------------------------------------------
// Diffeo pull-back metric: directional jet folded innermost-first.
__device__ __forceinline__ F3 accel_diffeo(const DevParams& P, F3 p, F3 y, float& valid) {
    if (P.n_stages == 1 && P.stages[0].kind == kStageTwist) {
        // Single twist (C4): J = [[R, b], [0, 1]] with R the rotation by z, so
        // J^-1 q = [R^T (q_xy - q_z b); q_z] and q_z = 0 for the twist:
        // a = -R^T (d0, d1) / det — the general fold below, specialised.
        // Expanding R^T (d0, d1) with cs^2 + sn^2 = det = 1 (diffeo.hpp:165-171)
        // the rotation cancels: a = (z'(2y' + z'x), z'(z'y - 2x'), 0), the
        // rotating-frame Coriolis + centrifugal terms.  No sincos, no
        // reciprocal; |det J| = 1 so the validity bound is unchanged.
        valid = fminf(valid, 1.f);
        return f3(y.z * fmaf(y.z, p.x, 2.f * y.y), y.z * fmaf(y.z, p.y, -2.f * y.x), 0.f);
    }
    float x0 = p.x, x1 = p.y, x2 = p.z;          // current point
    float w0 = y.x, w1 = y.y, w2 = y.z;          // J_inner y
    float q0 = 0.f, q1 = 0.f, q2 = 0.f;          // D^2 Phi_inner[y, y]
    float J[9] = {1.f, 0.f, 0.f, 0.f, 1.f, 0.f, 0.f, 0.f, 1.f};
    float vmin = 3.0e38f, dprod = 1.f;
    for (int s = 0; s < P.n_stages; ++s) {
        const DevStage& st = P.stages[s];
        float det;
        if (st.kind == kStageAffine) {                       // diffeo.hpp:133-141
            const float* m = st.v;
            const float n0 = m[0] * x0 + m[1] * x1 + m[2] * x2 + m[9];
            const float n1 = m[3] * x0 + m[4] * x1 + m[5] * x2 + m[10];
            const float n2 = m[6] * x0 + m[7] * x1 + m[8] * x2 + m[11];
            const float a0 = m[0] * q0 + m[1] * q1 + m[2] * q2;
            const float a1 = m[3] * q0 + m[4] * q1 + m[5] * q2;
            const float a2 = m[6] * q0 + m[7] * q1 + m[8] * q2;
            q0 = a0; q1 = a1; q2 = a2;
            const float b0 = m[0] * w0 + m[1] * w1 + m[2] * w2;
            const float b1 = m[3] * w0 + m[4] * w1 + m[5] * w2;
            const float b2 = m[6] * w0 + m[7] * w1 + m[8] * w2;
            w0 = b0; w1 = b1; w2 = b2;
            float R[9];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                R[c] = m[0] * J[c] + m[1] * J[3 + c] + m[2] * J[6 + c];
                R[3 + c] = m[3] * J[c] + m[4] * J[3 + c] + m[5] * J[6 + c];
                R[6 + c] = m[6] * J[c] + m[7] * J[3 + c] + m[8] * J[6 + c];
            }
#pragma unroll
            for (int k = 0; k < 9; ++k) J[k] = R[k];
            x0 = n0; x1 = n1; x2 = n2;
            det = st.det;
        } else if (st.kind == kStageTwist) {                 // diffeo.hpp:143-173
            float sn, cs;
#if RR_FAST_SINCOS
            __sincosf(x2, &sn, &cs);   // MUFU.SIN/COS: |z| <= ~10 in chart units
#else
            sincosf(x2, &sn, &cs);
#endif
            const float j02 = -(x0 * sn) - x1 * cs;          // d(image_0)/dz
            const float j12 = x0 * cs - x1 * sn;             // d(image_1)/dz
            // w^T H[0] w and w^T H[1] w (H[2] = 0)
            const float d0 = -w2 * (2.f * (w0 * sn + w1 * cs) + w2 * j12);
            const float d1 = w2 * (2.f * (w0 * cs - w1 * sn) + w2 * j02);
            const float a0 = d0 + cs * q0 - sn * q1 + j02 * q2;
            const float a1 = d1 + sn * q0 + cs * q1 + j12 * q2;
            q0 = a0; q1 = a1;
            const float b0 = cs * w0 - sn * w1 + j02 * w2;
            const float b1 = sn * w0 + cs * w1 + j12 * w2;
            w0 = b0; w1 = b1;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float r0 = cs * J[c] - sn * J[3 + c] + j02 * J[6 + c];
                const float r1 = sn * J[c] + cs * J[3 + c] + j12 * J[6 + c];
                J[c] = r0;
                J[3 + c] = r1;
            }
            x0 = j12;                                         // x c - y s
            x1 = -j02;                                        // x s + y c
            det = cs * cs + sn * sn;
        } else if (st.kind == kStageBend) {                   // EXTENSION (oracle/rro.c)
            const float k = st.v[0], c = st.v[1];
            float sn, cs;
            __sincosf(k * x0, &sn, &cs);
            const float yc = x1 - c;
            const float j00 = -k * cs * yc, j10 = -k * sn * yc;   // j01 = -sn, j11 = cs
            const float wxx = w0 * w0, wxy = 2.f * w0 * w1;
            const float d0 = wxx * (k * k * sn * yc) - wxy * (k * cs);
            const float d1 = -wxx * (k * k * cs * yc) - wxy * (k * sn);
            const float a0 = d0 + j00 * q0 - sn * q1;
            const float a1 = d1 + j10 * q0 + cs * q1;
            q0 = a0; q1 = a1;
            const float b0 = j00 * w0 - sn * w1;
            const float b1 = j10 * w0 + cs * w1;
            w0 = b0; w1 = b1;
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                const float r0 = j00 * J[cc] - sn * J[3 + cc];
                const float r1 = j10 * J[cc] + cs * J[3 + cc];
                J[cc] = r0;
                J[3 + cc] = r1;
            }
            x0 = -sn * yc;
            x1 = fmaf(cs, yc, c);
            det = -k * yc;
        } else {                                              // diffeo.hpp:175-193
            const float* b = st.v;
            const float ux = (x0 - b[0]) * b[3], uy = (x1 - b[1]) * b[4], uz = (x2 - b[2]) * b[5];
            const float e = b[6] * __expf(-0.5f * (ux * ux + uy * uy + uz * uz));
            const float gx = ux * b[3], gy = uy * b[4], gz = uz * b[5];   // grad f = -e g
            const float wg = w0 * gx + w1 * gy + w2 * gz;
            const float ws = w0 * w0 * b[3] * b[3] + w1 * w1 * b[4] * b[4] + w2 * w2 * b[5] * b[5];
            const float whw = e * (wg * wg - ws);                           // w^T Hess f w
            const float fq = -e * (gx * q0 + gy * q1 + gz * q2);          // grad f . q
            const float fw = -e * wg;                                       // grad f . w
            q0 = fmaf(b[7], whw + fq, q0);
            q1 = fmaf(b[8], whw + fq, q1);
            q2 = fmaf(b[9], whw + fq, q2);
            w0 = fmaf(b[7], fw, w0);
            w1 = fmaf(b[8], fw, w1);
            w2 = fmaf(b[9], fw, w2);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float r = -e * (gx * J[c] + gy * J[3 + c] + gz * J[6 + c]);
                J[c] = fmaf(b[7], r, J[c]);
                J[3 + c] = fmaf(b[8], r, J[3 + c]);
                J[6 + c] = fmaf(b[9], r, J[6 + c]);
            }
            x0 = fmaf(e, b[7], x0);
            x1 = fmaf(e, b[8], x1);
            x2 = fmaf(e, b[9], x2);
            det = 1.f - e * (b[7] * gx + b[8] * gy + b[9] * gz);
        }
        vmin = fminf(vmin, fabsf(det));
        dprod *= det;
        vmin = fminf(vmin, fabsf(dprod));
    }
    // a = -J^-1 q via the adjugate (linalg.hpp:223-236)
    const float c00 = J[4] * J[8] - J[5] * J[7];
    const float c01 = J[2] * J[7] - J[1] * J[8];
    const float c02 = J[1] * J[5] - J[2] * J[4];
    const float c10 = J[5] * J[6] - J[3] * J[8];
    const float c11 = J[0] * J[8] - J[2] * J[6];
    const float c12 = J[2] * J[3] - J[0] * J[5];
    const float c20 = J[3] * J[7] - J[4] * J[6];
    const float c21 = J[1] * J[6] - J[0] * J[7];
    const float c22 = J[0] * J[4] - J[1] * J[3];
    const float d = J[0] * c00 + J[1] * c10 + J[2] * c20;
    valid = fminf(valid, fminf(vmin, fabsf(d)));
    const float id = -rcp_approx(d);
    return f3(id * (c00 * q0 + c01 * q1 + c02 * q2), id * (c10 * q0 + c11 * q1 + c12 * q2),
              id * (c20 * q0 + c21 * q1 + c22 * q2));
}

// accel_diffeo for a ray pair (general chains; ray-pair kernel kDiffeoChain):
// the same directional-jet fold innermost-first with every per-ray operation
// packed (stage constants as broadcast pairs, DevStage::v2), sin/cos per ray,
// and the validity bound per ray.
__device__ __forceinline__ F2 neg2(F2 a) { return mul2(a, bc2(-1.f)); }

// State of the fold for a ray pair: the current point x, J_inner y (w),
// D^2 Phi_inner[y, y] (q) and the Jacobian J of the stages folded so far.
struct ChainX2 {
    F2 x0, x1, x2, w0, w1, w2, q0, q1, q2;
    F2 J[9];
};

// One stage of each kind; each returns the stage's det J (validity).
__device__ __forceinline__ F2 stage_affine_x2(const DevStage& st, ChainX2& c) {   // diffeo.hpp:133-141
    F2 m[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) m[k] = ld2(st.v2[k]);
    const F2 n0 = add2(fma2(m[2], c.x2, fma2(m[1], c.x1, mul2(m[0], c.x0))), m[9]);
    const F2 n1 = add2(fma2(m[5], c.x2, fma2(m[4], c.x1, mul2(m[3], c.x0))), m[10]);
    const F2 n2 = add2(fma2(m[8], c.x2, fma2(m[7], c.x1, mul2(m[6], c.x0))), m[11]);
    const F2 a0 = fma2(m[2], c.q2, fma2(m[1], c.q1, mul2(m[0], c.q0)));
    const F2 a1 = fma2(m[5], c.q2, fma2(m[4], c.q1, mul2(m[3], c.q0)));
    const F2 a2 = fma2(m[8], c.q2, fma2(m[7], c.q1, mul2(m[6], c.q0)));
    c.q0 = a0; c.q1 = a1; c.q2 = a2;
    const F2 b0 = fma2(m[2], c.w2, fma2(m[1], c.w1, mul2(m[0], c.w0)));
    const F2 b1 = fma2(m[5], c.w2, fma2(m[4], c.w1, mul2(m[3], c.w0)));
    const F2 b2 = fma2(m[8], c.w2, fma2(m[7], c.w1, mul2(m[6], c.w0)));
    c.w0 = b0; c.w1 = b1; c.w2 = b2;
    F2 R[9];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        R[k] = fma2(m[2], c.J[6 + k], fma2(m[1], c.J[3 + k], mul2(m[0], c.J[k])));
        R[3 + k] = fma2(m[5], c.J[6 + k], fma2(m[4], c.J[3 + k], mul2(m[3], c.J[k])));
        R[6 + k] = fma2(m[8], c.J[6 + k], fma2(m[7], c.J[3 + k], mul2(m[6], c.J[k])));
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) c.J[k] = R[k];
    c.x0 = n0; c.x1 = n1; c.x2 = n2;
    return ld2(st.det2);
}

__device__ __forceinline__ F2 stage_twist_x2(ChainX2& c) {                        // diffeo.hpp:143-173
    float sa, ca, sb, cb;
    __sincosf(lo2(c.x2), &sa, &ca);
    __sincosf(hi2(c.x2), &sb, &cb);
    const F2 sn = mk2(sa, sb), cs = mk2(ca, cb);
    const F2 j02 = neg2(fma2(c.x1, cs, mul2(c.x0, sn)));            // d(image_0)/dz
    const F2 j12 = fnma2(c.x1, sn, mul2(c.x0, cs));                 // d(image_1)/dz
    const F2 two = bc2(2.f);
    // w^T H[0] w and w^T H[1] w (H[2] = 0)
    const F2 d0 = neg2(mul2(c.w2, fma2(two, fma2(c.w1, cs, mul2(c.w0, sn)), mul2(c.w2, j12))));
    const F2 d1 = mul2(c.w2, fma2(two, fnma2(c.w1, sn, mul2(c.w0, cs)), mul2(c.w2, j02)));
    const F2 a0 = fma2(j02, c.q2, fnma2(sn, c.q1, fma2(cs, c.q0, d0)));
    const F2 a1 = fma2(j12, c.q2, fma2(cs, c.q1, fma2(sn, c.q0, d1)));
    c.q0 = a0; c.q1 = a1;
    const F2 b0 = fma2(j02, c.w2, fnma2(sn, c.w1, mul2(cs, c.w0)));
    const F2 b1 = fma2(j12, c.w2, fma2(cs, c.w1, mul2(sn, c.w0)));
    c.w0 = b0; c.w1 = b1;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const F2 r0 = fma2(j02, c.J[6 + k], fnma2(sn, c.J[3 + k], mul2(cs, c.J[k])));
        const F2 r1 = fma2(j12, c.J[6 + k], fma2(cs, c.J[3 + k], mul2(sn, c.J[k])));
        c.J[k] = r0;
        c.J[3 + k] = r1;
    }
    c.x0 = j12;                                                     // x c - y s
    c.x1 = neg2(j02);                                               // x s + y c
    return fma2(sn, sn, mul2(cs, cs));
}

__device__ __forceinline__ F2 stage_bend_x2(const DevStage& st, ChainX2& c) {     // EXTENSION (oracle/rro.c)
    const F2 k = ld2(st.v2[0]), cc = ld2(st.v2[1]);
    const F2 kx = mul2(k, c.x0);
    float sa, ca, sb, cb;
    __sincosf(lo2(kx), &sa, &ca);
    __sincosf(hi2(kx), &sb, &cb);
    const F2 sn = mk2(sa, sb), cs = mk2(ca, cb);
    const F2 yc = sub2(c.x1, cc);
    const F2 kcs = mul2(k, cs), ksn = mul2(k, sn);
    const F2 j00 = neg2(mul2(kcs, yc)), j10 = neg2(mul2(ksn, yc));   // j01 = -sn, j11 = cs
    const F2 wxx = mul2(c.w0, c.w0), wxy = mul2(bc2(2.f), mul2(c.w0, c.w1));
    const F2 d0 = fnma2(wxy, kcs, mul2(wxx, mul2(mul2(k, ksn), yc)));
    const F2 d1 = neg2(fma2(wxy, ksn, mul2(wxx, mul2(mul2(k, kcs), yc))));
    const F2 a0 = fnma2(sn, c.q1, fma2(j00, c.q0, d0));
    const F2 a1 = fma2(cs, c.q1, fma2(j10, c.q0, d1));
    c.q0 = a0; c.q1 = a1;
    const F2 b0 = fnma2(sn, c.w1, mul2(j00, c.w0));
    const F2 b1 = fma2(cs, c.w1, mul2(j10, c.w0));
    c.w0 = b0; c.w1 = b1;
#pragma unroll
    for (int m = 0; m < 3; ++m) {
        const F2 r0 = fnma2(sn, c.J[3 + m], mul2(j00, c.J[m]));
        const F2 r1 = fma2(cs, c.J[3 + m], mul2(j10, c.J[m]));
        c.J[m] = r0;
        c.J[3 + m] = r1;
    }
    c.x0 = neg2(mul2(sn, yc));
    c.x1 = fma2(cs, yc, cc);
    return neg2(mul2(k, yc));
}

__device__ __forceinline__ F2 stage_bump_x2(const DevStage& st, ChainX2& c) {     // diffeo.hpp:175-193
    const F2 cx = ld2(st.v2[0]), cy = ld2(st.v2[1]), cz = ld2(st.v2[2]);
    const F2 sx = ld2(st.v2[3]), sy = ld2(st.v2[4]), sz = ld2(st.v2[5]);
    const F2 amp = ld2(st.v2[6]), dx = ld2(st.v2[7]), dy = ld2(st.v2[8]), dz = ld2(st.v2[9]);
    const F2 ux = mul2(sub2(c.x0, cx), sx), uy = mul2(sub2(c.x1, cy), sy), uz = mul2(sub2(c.x2, cz), sz);
    const F2 uu = fma2(uz, uz, fma2(uy, uy, mul2(ux, ux)));
    const F2 ee = mul2(bc2(-0.5f), uu);
    const F2 e = mul2(amp, mk2(__expf(lo2(ee)), __expf(hi2(ee))));
    const F2 gx = mul2(ux, sx), gy = mul2(uy, sy), gz = mul2(uz, sz);   // grad f = -e g
    const F2 wg = fma2(c.w2, gz, fma2(c.w1, gy, mul2(c.w0, gx)));
    const F2 ws = fma2(mul2(c.w2, c.w2), mul2(sz, sz),
                       fma2(mul2(c.w1, c.w1), mul2(sy, sy), mul2(mul2(c.w0, c.w0), mul2(sx, sx))));
    const F2 whw = mul2(e, fnma2(bc2(1.f), ws, mul2(wg, wg)));         // w^T Hess f w
    const F2 fq = neg2(mul2(e, fma2(gz, c.q2, fma2(gy, c.q1, mul2(gx, c.q0)))));   // grad f . q
    const F2 fw = neg2(mul2(e, wg));                                  // grad f . w
    const F2 hq = add2(whw, fq);
    c.q0 = fma2(dx, hq, c.q0);
    c.q1 = fma2(dy, hq, c.q1);
    c.q2 = fma2(dz, hq, c.q2);
    c.w0 = fma2(dx, fw, c.w0);
    c.w1 = fma2(dy, fw, c.w1);
    c.w2 = fma2(dz, fw, c.w2);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const F2 r = neg2(mul2(e, fma2(gz, c.J[6 + k], fma2(gy, c.J[3 + k], mul2(gx, c.J[k])))));
        c.J[k] = fma2(dx, r, c.J[k]);
        c.J[3 + k] = fma2(dy, r, c.J[3 + k]);
        c.J[6 + k] = fma2(dz, r, c.J[6 + k]);
    }
    c.x0 = fma2(e, dx, c.x0);
    c.x1 = fma2(e, dy, c.x1);
    c.x2 = fma2(e, dz, c.x2);
    return fnma2(e, fma2(dz, gz, fma2(dy, gy, mul2(dx, gx))), bc2(1.f));
}

template <int KS>
__device__ __forceinline__ F2 stage_x2(const DevStage& st, ChainX2& c) {
    if constexpr (KS == kStageAffine) return stage_affine_x2(st, c);
    else if constexpr (KS == kStageTwist) return stage_twist_x2(c);
    else if constexpr (KS == kStageBend) return stage_bend_x2(st, c);
    else return stage_bump_x2(st, c);
}

// Compile-time chain signatures (the kDiffeoChain kernel's NB template
// argument): 0 = any chain, folded by a run-time loop over the stage kinds;
// otherwise n | kind_0 << 4 | kind_1 << 8 | ... (innermost stage first), the
// fold unrolled with every stage's kind known to the compiler (no kind
// switch, no phi moves of the fold state at its joins).
constexpr int chain_sig2(int k0, int k1) { return 2 | (k0 << 4) | (k1 << 8); }
constexpr int sig_len(int sig) { return sig & 15; }
constexpr int sig_kind(int sig, int i) { return (sig >> (4 + 4 * i)) & 15; }

template <int SIG, int I>
__device__ __forceinline__ void fold_static_x2(const DevParams& P, ChainX2& c, float (&vmin)[2],
                                               float (&dprod)[2]) {
    if constexpr (I < sig_len(SIG)) {
        const F2 det = stage_x2<sig_kind(SIG, I)>(P.stages[I], c);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const float dt = get2(det, r);
            vmin[r] = fminf(vmin[r], fabsf(dt));
            dprod[r] *= dt;
            vmin[r] = fminf(vmin[r], fabsf(dprod[r]));
        }
        fold_static_x2<SIG, I + 1>(P, c, vmin, dprod);
    }
}

template <int SIG = 0>
__device__ __forceinline__ P3 accel_diffeo_x2(const DevParams& P, const P3& p, const P3& y,
                                              float (&valid)[2]) {
    ChainX2 c{p.x, p.y, p.z, y.x, y.y, y.z, bc2(0.f), bc2(0.f), bc2(0.f),
              {bc2(1.f), bc2(0.f), bc2(0.f), bc2(0.f), bc2(1.f), bc2(0.f), bc2(0.f), bc2(0.f), bc2(1.f)}};
    float vmin[2] = {3.0e38f, 3.0e38f}, dprod[2] = {1.f, 1.f};
    if constexpr (SIG != 0) {
        fold_static_x2<SIG, 0>(P, c, vmin, dprod);
    } else {
        for (int s = 0; s < P.n_stages; ++s) {
            const DevStage& st = P.stages[s];
            F2 det;
            if (st.kind == kStageAffine) det = stage_affine_x2(st, c);
            else if (st.kind == kStageTwist) det = stage_twist_x2(c);
            else if (st.kind == kStageBend) det = stage_bend_x2(st, c);
            else det = stage_bump_x2(st, c);
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const float dt = get2(det, r);
                vmin[r] = fminf(vmin[r], fabsf(dt));
                dprod[r] *= dt;
                vmin[r] = fminf(vmin[r], fabsf(dprod[r]));
            }
        }
    }
    const F2 q0 = c.q0, q1 = c.q1, q2 = c.q2;
    const F2 (&J)[9] = c.J;
    // a = -J^-1 q via the adjugate (linalg.hpp:223-236)
    const F2 c00 = fnma2(J[5], J[7], mul2(J[4], J[8]));
    const F2 c01 = fnma2(J[1], J[8], mul2(J[2], J[7]));
    const F2 c02 = fnma2(J[2], J[4], mul2(J[1], J[5]));
    const F2 c10 = fnma2(J[3], J[8], mul2(J[5], J[6]));
    const F2 c11 = fnma2(J[2], J[6], mul2(J[0], J[8]));
    const F2 c12 = fnma2(J[0], J[5], mul2(J[2], J[3]));
    const F2 c20 = fnma2(J[4], J[6], mul2(J[3], J[7]));
    const F2 c21 = fnma2(J[0], J[7], mul2(J[1], J[6]));
    const F2 c22 = fnma2(J[1], J[3], mul2(J[0], J[4]));
    const F2 d = fma2(J[2], c20, fma2(J[1], c10, mul2(J[0], c00)));
#pragma unroll
    for (int r = 0; r < 2; ++r) valid[r] = fminf(valid[r], fminf(vmin[r], fabsf(get2(d, r))));
    const F2 id = neg2(mk2(rcp_approx(lo2(d)), rcp_approx(hi2(d))));
    return P3{mul2(id, fma2(c02, q2, fma2(c01, q1, mul2(c00, q0)))),
              mul2(id, fma2(c12, q2, fma2(c11, q1, mul2(c10, q0)))),
              mul2(id, fma2(c22, q2, fma2(c21, q1, mul2(c20, q0))))};
}

template <int KIND, int NB>
__device__ __forceinline__ F3 accel(const DevParams& P, uint32_t um, F3 p, F3 y, float& valid) {
    if constexpr (KIND == kEuclid) {
        return f3(0.f, 0.f, 0.f);
    } else if constexpr (KIND == kBumps) {
        return accel_bumps<NB>(P, um, p, y);
    } else if constexpr (KIND == kGraphGeneral) {
        return accel_graph_general(P, p, y);
    } else {
        return accel_diffeo(P, p, y, valid);
    }
}

// ---------------------------------------------------------------------------
// Chord-vs-primitive intersection (scene.cpp:15-109), FP32.
__device__ __forceinline__ bool slab(float a, float d, float lo, float hi, float& smin, float& smax) {
    if (d == 0.f) return !(a < lo || a > hi);
    float s1 = (lo - a) / d;
    float s2 = (hi - a) / d;
    if (s1 > s2) {
        const float t = s1;
        s1 = s2;
        s2 = t;
    }
    smin = fmaxf(smin, s1);
    smax = fminf(smax, s2);
    return !(smin > smax);
}

// chord_box_entry (scene.cpp:15-34) for a box given per axis.
__device__ __forceinline__ bool chord_box_entry(F3 a, F3 d, F3 lo, F3 hi, float& s_out) {
    float smin = 0.f, smax = 1.f;
    if (!slab(a.x, d.x, lo.x, hi.x, smin, smax)) return false;
    if (!slab(a.y, d.y, lo.y, hi.y, smin, smax)) return false;
    if (!slab(a.z, d.z, lo.z, hi.z, smin, smax)) return false;
    s_out = smin;
    return true;
}

__device__ __forceinline__ float comp(F3 v, int i) { return i == 0 ? v.x : (i == 1 ? v.y : v.z); }
__device__ __forceinline__ void set_comp(F3& v, int i, float x) {
    if (i == 0) v.x = x;
    else if (i == 1) v.y = x;
    else v.z = x;
}

// hit_grid (scene.cpp:36-54): slabs around x_dim = k*spacing clipped to bounds.
template <int DIM>
__device__ __forceinline__ void hit_grid_dim(const DevGrid& g, F3 a, F3 b, F3 d, bool& have,
                                             float& best) {
    const float ad = comp(a, DIM), bd = comp(b, DIM);
    const float clo = fminf(ad, bd), chi = fmaxf(ad, bd);
    const int kmin = (int)ceilf((clo - g.hw) / g.spacing);
    const int kmax = (int)floorf((chi + g.hw) / g.spacing);
    for (int k = kmin; k <= kmax; ++k) {
        F3 lo = f3(g.lo[0], g.lo[1], g.lo[2]), hi = f3(g.hi[0], g.hi[1], g.hi[2]);
        const float plane = (float)k * g.spacing;
        set_comp(lo, DIM, fmaxf(comp(lo, DIM), plane - g.hw));
        set_comp(hi, DIM, fminf(comp(hi, DIM), plane + g.hw));
        if (comp(lo, DIM) > comp(hi, DIM)) continue;
        float s;
        if (chord_box_entry(a, d, lo, hi, s) && (!have || s < best)) {
            best = s;
            have = true;
        }
    }
}

__device__ __forceinline__ bool hit_grid(const DevGrid& g, F3 a, F3 b, F3 d, float& s_out) {
    bool have = false;
    float best = 0.f;
    hit_grid_dim<0>(g, a, b, d, have, best);
    hit_grid_dim<1>(g, a, b, d, have, best);
    hit_grid_dim<2>(g, a, b, d, have, best);
    s_out = best;
    return have;
}

// hit_sphere (scene.cpp:56-71) with a conservative early-out: a chord of
// length L starting outside cannot reach the sphere when |oc| > r + L, i.e.
// c = |oc|^2 - r^2 > (2r + L) L.
__device__ __forceinline__ bool hit_sphere(const DevSphere& sp, F3 a, F3 d, float qa, float len,
                                           float& s_out) {
    const float ox = a.x - sp.c[0], oy = a.y - sp.c[1], oz = a.z - sp.c[2];
    const float c = fmaf(ox, ox, fmaf(oy, oy, fmaf(oz, oz, -sp.r2)));
    if (c <= 0.f) {
        s_out = 0.f;
        return true;
    }
    if (fmaf(-len, sp.two_r + len, c) > 0.f) return false;
    const float qb = 2.f * (ox * d.x + oy * d.y + oz * d.z);
    if (qb >= 0.f) return false;
    const float disc = qb * qb - 4.f * qa * c;
    if (disc < 0.f) return false;
    const float q = 0.5f * (sqrtf(disc) - qb);
    const float s = c / q;
    if (s > 1.f) return false;
    s_out = s;
    return true;
}

__device__ __forceinline__ bool hit_half_space(const DevHalf& hs, F3 a, F3 d, float& s_out) {
    const float e0 = hs.n[0] * a.x + hs.n[1] * a.y + hs.n[2] * a.z - hs.off;
    if (e0 <= 0.f) {
        s_out = 0.f;
        return true;
    }
    const float de = hs.n[0] * d.x + hs.n[1] * d.y + hs.n[2] * d.z;
    if (de >= 0.f) return false;
    const float s = -e0 / de;
    if (s > 1.f) return false;
    s_out = s;
    return true;
}

// ---------------------------------------------------------------------------
// EXTENSION: triangle meshes.  The chord [a, b] of a step is tested against a
// BVH (slab test per node, Moller-Trumbore per triangle, ties keep the lower
// original triangle index: oracle/rro.c hit_mesh).  Each lane also keeps a
// "free distance": the distance from a query point to the nearest leaf box;
// while the marched path stays inside that ball (sum of chord lengths) no
// mesh test is needed.  Both are __noinline__ so scenes without meshes keep
// the march loop's register allocation.
__device__ __forceinline__ bool mesh_chord_impl(const DevMesh& M, F3 a, F3 d, float& best_s, int& best_rec) {
    const float ix = d.x != 0.f ? 1.f / d.x : 3.0e38f;
    const float iy = d.y != 0.f ? 1.f / d.y : 3.0e38f;
    const float iz = d.z != 0.f ? 1.f / d.z : 3.0e38f;
    bool have = false;
    float best = 1.f;
    int best_t = 0x7fffffff;
    int stack[64];
    int sp = 0, node = 0;
    for (;;) {
        const float4 n0 = __ldg(M.nodes + 2 * node), n1 = __ldg(M.nodes + 2 * node + 1);
        float t0 = 0.f, t1 = best;
        {
            float u = (n0.x - a.x) * ix, w = (n1.x - a.x) * ix;
            t0 = fmaxf(t0, fminf(u, w));
            t1 = fminf(t1, fmaxf(u, w));
            u = (n0.y - a.y) * iy;
            w = (n1.y - a.y) * iy;
            t0 = fmaxf(t0, fminf(u, w));
            t1 = fminf(t1, fmaxf(u, w));
            u = (n0.z - a.z) * iz;
            w = (n1.z - a.z) * iz;
            t0 = fmaxf(t0, fminf(u, w));
            t1 = fminf(t1, fmaxf(u, w));
        }
        // a zero chord component makes u, w +-inf or NaN: fall back to the
        // containment test on that axis
        bool overlap = t0 <= t1;
        if (d.x == 0.f) overlap = overlap && a.x >= n0.x && a.x <= n1.x;
        if (d.y == 0.f) overlap = overlap && a.y >= n0.y && a.y <= n1.y;
        if (d.z == 0.f) overlap = overlap && a.z >= n0.z && a.z <= n1.z;
        if (overlap) {
            const int first = __float_as_int(n0.w), cnt = __float_as_int(n1.w);
            if (cnt > 0) {
                for (int i = first; i < first + cnt; ++i) {
                    const float4 r0 = __ldg(M.tris + 3 * i), r1 = __ldg(M.tris + 3 * i + 1),
                                 r2 = __ldg(M.tris + 3 * i + 2);
                    const F3 e1 = f3(r1.x, r1.y, r1.z), e2 = f3(r2.x, r2.y, r2.z);
                    const F3 pv = f3(d.y * e2.z - d.z * e2.y, d.z * e2.x - d.x * e2.z, d.x * e2.y - d.y * e2.x);
                    const float det = e1.x * pv.x + e1.y * pv.y + e1.z * pv.z;
                    if (det == 0.f) continue;
                    const float inv = 1.f / det;
                    const F3 tv = f3(a.x - r0.x, a.y - r0.y, a.z - r0.z);
                    const float u = (tv.x * pv.x + tv.y * pv.y + tv.z * pv.z) * inv;
                    if (u < 0.f || u > 1.f) continue;
                    const F3 qv = f3(tv.y * e1.z - tv.z * e1.y, tv.z * e1.x - tv.x * e1.z, tv.x * e1.y - tv.y * e1.x);
                    const float v = (d.x * qv.x + d.y * qv.y + d.z * qv.z) * inv;
                    if (v < 0.f || u + v > 1.f) continue;
                    const float s = (e2.x * qv.x + e2.y * qv.y + e2.z * qv.z) * inv;
                    if (s < 0.f || s > 1.f) continue;
                    const int t = __float_as_int(r0.w);
                    if (!have || s < best || (s == best && t < best_t)) {
                        best = s;
                        best_t = t;
                        best_rec = i;
                        have = true;
                    }
                }
            } else if (sp < 63) {
                stack[sp++] = first;      // right child
                node = node + 1;          // left child
                continue;
            }
        }
        if (sp == 0) break;
        node = stack[--sp];
    }
    if (have) best_s = best;
    return have;
}

__device__ __forceinline__ float box_dist2(float4 n0, float4 n1, F3 p) {
    const float dx = fmaxf(fmaxf(n0.x - p.x, p.x - n1.x), 0.f);
    const float dy = fmaxf(fmaxf(n0.y - p.y, p.y - n1.y), 0.f);
    const float dz = fmaxf(fmaxf(n0.z - p.z, p.z - n1.z), 0.f);
    return fmaf(dx, dx, fmaf(dy, dy, dz * dz));
}

// Distance from p to the nearest leaf box (capped): no triangle lies closer.
// Nearest-child-first descent so the bound tightens early.
#ifndef RR_DIFFEO_RK4_UNROLL
#define RR_DIFFEO_RK4_UNROLL 0   // general diffeo chains: 1 = RK4 stages unrolled (4 copies of the fold);
                                 // rolled is faster (I-cache: bend 58.0 -> 50.5 ms, profiles/r1k_unroll_ab.log)
#endif
#ifndef RR_TWIST_RK4
#define RR_TWIST_RK4 1     // z-free RK4 for a single-twist metric (march_fixed)
#endif
#ifndef RR_TWIST_XY_PAIRS
// one-ray twist RK4 with the (x, y) components of the ray packed as FFMA2
// pairs: C4 twist + 100k mesh 10.17 -> 9.35 ms (profiles/r2s_twist_xy_ab.log)
#define RR_TWIST_XY_PAIRS 1
#endif
#ifndef RR_MESH_FREE_CAP
#define RR_MESH_FREE_CAP 0.5f   // re-measured with rolled diffeo stages + 6 CTAs/SM (profiles/r1k_freecap_ab.log):
                                // caps 0.25 / 0.5 / 1 / 2: C4 twist 13.0 / 12.8 / 13.3 / 14.2 ms, twist+bend 50.7 / 50.5 / 51.1 / 51.5 ms
#endif
__device__ __forceinline__ float mesh_free_impl(const DevMesh& M, F3 p, float cap) {
    float best2 = cap * cap;
    int stack[48];
    float sd[48];
    int sp = 0, node = 0;
    float nd2 = box_dist2(__ldg(M.nodes), __ldg(M.nodes + 1), p);
    for (;;) {
        if (nd2 < best2) {
            const float4 n0 = __ldg(M.nodes + 2 * node), n1 = __ldg(M.nodes + 2 * node + 1);
            if (__float_as_int(n1.w) > 0) {
                best2 = nd2;
            } else {
                const int l = node + 1, r = __float_as_int(n0.w);
                const float dl = box_dist2(__ldg(M.nodes + 2 * l), __ldg(M.nodes + 2 * l + 1), p);
                const float dr = box_dist2(__ldg(M.nodes + 2 * r), __ldg(M.nodes + 2 * r + 1), p);
                const bool lf = dl <= dr;
                if (sp < 48) {
                    stack[sp] = lf ? r : l;
                    sd[sp] = lf ? dr : dl;
                    ++sp;
                }
                node = lf ? l : r;
                nd2 = lf ? dl : dr;
                continue;
            }
        }
        // pop the next candidate that can still beat the bound
        bool found = false;
        while (sp > 0) {
            --sp;
            if (sd[sp] < best2) {
                node = stack[sp];
                nd2 = sd[sp];
                found = true;
                break;
            }
        }
        if (!found) break;
    }
    return sqrtf(best2);
}

__device__ __noinline__ bool mesh_chord(const DevMesh& M, F3 a, F3 d, float& best_s, int& best_rec) {
    return mesh_chord_impl(M, a, d, best_s, best_rec);
}
__device__ __noinline__ float mesh_free(const DevMesh& M, F3 p, float cap) {
    return mesh_free_impl(M, p, cap);
}

// Free distance of point a from every mesh by its distance grid: a lower
// bound of the distance from a to any triangle (0 outside the grid or next
// to the mesh).  One byte load per mesh instead of a nearest-first BVH query.
__device__ __forceinline__ float mesh_grid_free(const DevParams& P, F3 a) {
    float fr = 3.0e38f;
    for (int i = 0; i < P.n_meshes; ++i) {
        const DevMesh& M = P.meshes[i];
        if (M.dG == 0) return 0.f;
        const float fx = (a.x - M.dlo[0]) * M.dinv[0], fy = (a.y - M.dlo[1]) * M.dinv[1];
        const float fz = (a.z - M.dlo[2]) * M.dinv[2];
        const float g = (float)M.dG;
        if (!(fx >= 0.f && fy >= 0.f && fz >= 0.f && fx < g && fy < g && fz < g)) return 0.f;
        const unsigned cell = ((unsigned)fz * M.dG + (unsigned)fy) * M.dG + (unsigned)fx;
        fr = fminf(fr, (float)__ldg(M.dist + cell) * M.dq);
    }
    return fr;
}

// Nearest hit over all primitives; ties keep the lower primitive index
// (scene.cpp:99-109), i.e. the lexicographic minimum of (s, index).
__device__ __forceinline__ bool consider(bool h, float s, int idx, int id, bool& have, float& best,
                                         int& prim, int& hid) {
    if (h && (!have || s < best || (s == best && idx < prim))) {
        best = s;
        prim = idx;
        hid = id;   // (kind << 8) | slot, for the hit normal (EXT shading)
        have = true;
        return true;
    }
    return false;
}

// Free-distance budget of the analytic primitives (spheres, half-spaces):
// `sfree` is a lower bound of the distance from the current chord start to
// every sphere and half-space region.  A chord of length len < sfree cannot
// reach any of them (so the exact tests could only report "no hit"); the
// budget shrinks by len per skipped chord and is recomputed at the chord end
// after every tested chord.  Inside-start chords have sfree <= 0 and are
// always tested.  Results are identical to testing every chord.
__device__ __forceinline__ float analytic_free(const DevParams& P, F3 b) {
    float fr = 3.0e38f;
#pragma unroll
    for (int i = 0; i < kStaticSpheres; ++i)
        if (i < P.n_spheres) {
            const DevSphere& sp = P.spheres[i];
            const float ox = b.x - sp.c[0], oy = b.y - sp.c[1], oz = b.z - sp.c[2];
            fr = fminf(fr, sqrt_approx(fmaf(ox, ox, fmaf(oy, oy, oz * oz))) - sp.r);
        }
    for (int i = kStaticSpheres; i < P.n_spheres; ++i) {
        const DevSphere& sp = P.spheres[i];
        const float ox = b.x - sp.c[0], oy = b.y - sp.c[1], oz = b.z - sp.c[2];
        fr = fminf(fr, sqrt_approx(fmaf(ox, ox, fmaf(oy, oy, oz * oz))) - sp.r);
    }
#pragma unroll
    for (int i = 0; i < kStaticHalves; ++i)
        if (i < P.n_halves) {
            const DevHalf& hs = P.halves[i];
            fr = fminf(fr, (fmaf(hs.n[0], b.x, fmaf(hs.n[1], b.y, hs.n[2] * b.z)) - hs.off) * hs.inv_norm);
        }
    for (int i = kStaticHalves; i < P.n_halves; ++i) {
        const DevHalf& hs = P.halves[i];
        fr = fminf(fr, (fmaf(hs.n[0], b.x, fmaf(hs.n[1], b.y, hs.n[2] * b.z)) - hs.off) * hs.inv_norm);
    }
    // rounding margin of the FP32 distances (approximate sqrt, world units)
    return fr - fmaf(2e-6f, fabsf(fr), 1e-5f) - 1e-6f * (fabsf(b.x) + fabsf(b.y) + fabsf(b.z));
}

template <bool MESH>
__device__ __forceinline__ bool intersect(const DevParams& P, F3 a, F3 b, float& s_best,
                                          int& prim, int& hid, float& mfree, int& mrec,
                                          float& sfree, float& clen) {
    const F3 d = f3(b.x - a.x, b.y - a.y, b.z - a.z);
    const float qa = fmaf(d.x, d.x, fmaf(d.y, d.y, d.z * d.z));
    const float len = fmaf(sqrt_approx(qa), 1.0001f, 1e-30f);   // conservative chord length
    clen = len;
    bool have = false;
    float s = 0.f;
    if (len < sfree) {
        sfree -= len;                     // no sphere / half-space within reach
    } else {
#pragma unroll
        for (int i = 0; i < kStaticSpheres; ++i)
            if (i < P.n_spheres) {
                const bool h = hit_sphere(P.spheres[i], a, d, qa, len, s);
                consider(h, s, P.spheres[i].index, (kPrimSphere << 8) | i, have, s_best, prim, hid);
            }
        for (int i = kStaticSpheres; i < P.n_spheres; ++i) {
            const bool h = hit_sphere(P.spheres[i], a, d, qa, len, s);
            consider(h, s, P.spheres[i].index, (kPrimSphere << 8) | i, have, s_best, prim, hid);
        }
#pragma unroll
        for (int i = 0; i < kStaticHalves; ++i)
            if (i < P.n_halves) {
                const bool h = hit_half_space(P.halves[i], a, d, s);
                consider(h, s, P.halves[i].index, (kPrimHalfSpace << 8) | i, have, s_best, prim, hid);
            }
        for (int i = kStaticHalves; i < P.n_halves; ++i) {
            const bool h = hit_half_space(P.halves[i], a, d, s);
            consider(h, s, P.halves[i].index, (kPrimHalfSpace << 8) | i, have, s_best, prim, hid);
        }
        if (!have) sfree = analytic_free(P, b);
    }
    for (int i = 0; i < P.n_grids; ++i) {
        const bool h = hit_grid(P.grids[i], a, b, d, s);
        consider(h, s, P.grids[i].index, (kPrimGrid << 8) | i, have, s_best, prim, hid);
    }
    if (MESH) {
        float gd;
        if (len < mfree) {
            mfree -= len;                 // the chord stays inside the free ball
        } else if ((gd = mesh_grid_free(P, a)) > len) {
            mfree = gd - len;             // inside the distance grid's free ball around a
        } else {
            for (int i = 0; i < P.n_meshes; ++i) {
                int rec = 0;
                const bool h = mesh_chord(P.meshes[i], a, d, s, rec);
                if (consider(h, s, P.meshes[i].index, (kPrimMesh << 8) | i, have, s_best, prim, hid))
                    mrec = rec;
            }
            float fr = 3.0e38f;
            for (int i = 0; i < P.n_meshes; ++i) fr = fminf(fr, mesh_free(P.meshes[i], b, RR_MESH_FREE_CAP));
            mfree = fr;
        }
    }
    return have;
}

template <bool MESH>
__device__ __forceinline__ bool intersect(const DevParams& P, F3 a, F3 b, float& s_best,
                                          int& prim, int& hid, float& mfree, int& mrec,
                                          float& sfree) {
    float clen;
    return intersect<MESH>(P, a, b, s_best, prim, hid, mfree, mrec, sfree, clen);
}

// Outward unit normal of a hit (EXTENSION shading; oracle/rro.c
// intersect_segment_n): sphere radial, half-space n/|n|, grid entry face,
// -chord direction for a chord that starts inside (s == 0).
__device__ F3 hit_normal(const DevParams& P, int hid, float s, F3 a, F3 b, F3 point, int mrec) {
    const F3 d = f3(b.x - a.x, b.y - a.y, b.z - a.z);
    if (hid >> 8 == kPrimMesh) {                // geometric normal facing the chord
        const DevMesh& M = P.meshes[hid & 0xff];
        const float4 r1 = __ldg(M.tris + 3 * mrec + 1), r2 = __ldg(M.tris + 3 * mrec + 2);
        F3 n = f3(r1.y * r2.z - r1.z * r2.y, r1.z * r2.x - r1.x * r2.z, r1.x * r2.y - r1.y * r2.x);
        const float sg = (n.x * d.x + n.y * d.y + n.z * d.z) > 0.f ? -1.f : 1.f;
        const float il = sg * rsqrtf(n.x * n.x + n.y * n.y + n.z * n.z);
        return f3(n.x * il, n.y * il, n.z * il);
    }
    const float kind = hid >> 8;
    const int slot = hid & 0xff;
    F3 n;
    int grid_axis = -1;
    if (s > 0.f && hid >> 8 == kPrimGrid) {
        // re-run the winning slab entry with axis tracking
        const DevGrid& g = P.grids[slot];
        float best = 2.f;
        const float av[3] = {a.x, a.y, a.z}, bv[3] = {b.x, b.y, b.z}, dv[3] = {d.x, d.y, d.z};
        for (int dim = 0; dim < 3; ++dim) {
            const float clo = fminf(av[dim], bv[dim]), chi = fmaxf(av[dim], bv[dim]);
            const int kmin = (int)ceilf((clo - g.hw) / g.spacing);
            const int kmax = (int)floorf((chi + g.hw) / g.spacing);
            for (int k = kmin; k <= kmax; ++k) {
                float lo[3] = {g.lo[0], g.lo[1], g.lo[2]}, hi[3] = {g.hi[0], g.hi[1], g.hi[2]};
                const float plane = (float)k * g.spacing;
                lo[dim] = fmaxf(lo[dim], plane - g.hw);
                hi[dim] = fminf(hi[dim], plane + g.hw);
                if (lo[dim] > hi[dim]) continue;
                float smin = 0.f, smax = 1.f;
                int ax = -1;
                bool ok = true;
                for (int e = 0; e < 3 && ok; ++e) {
                    if (dv[e] == 0.f) {
                        ok = !(av[e] < lo[e] || av[e] > hi[e]);
                        continue;
                    }
                    float s1 = (lo[e] - av[e]) / dv[e], s2 = (hi[e] - av[e]) / dv[e];
                    if (s1 > s2) {
                        const float t = s1;
                        s1 = s2;
                        s2 = t;
                    }
                    if (s1 > smin) {
                        smin = s1;
                        ax = e;
                    }
                    smax = fminf(smax, s2);
                    ok = !(smin > smax);
                }
                if (ok && smin < best) {
                    best = smin;
                    grid_axis = ax;
                }
            }
        }
    }
    (void)kind;
    if (s == 0.f || (hid >> 8 == kPrimGrid && grid_axis < 0)) {
        const float il = rsqrtf(fmaxf(d.x * d.x + d.y * d.y + d.z * d.z, 1e-30f));
        n = f3(-d.x * il, -d.y * il, -d.z * il);
    } else if (hid >> 8 == kPrimSphere) {
        const DevSphere& sp = P.spheres[slot];
        const F3 r = f3(point.x - sp.c[0], point.y - sp.c[1], point.z - sp.c[2]);
        const float il = rsqrtf(r.x * r.x + r.y * r.y + r.z * r.z);
        n = f3(r.x * il, r.y * il, r.z * il);
    } else if (hid >> 8 == kPrimHalfSpace) {
        const DevHalf& hs = P.halves[slot];
        const float il = rsqrtf(hs.n[0] * hs.n[0] + hs.n[1] * hs.n[1] + hs.n[2] * hs.n[2]);
        n = f3(hs.n[0] * il, hs.n[1] * il, hs.n[2] * il);
    } else {
        const float dc = grid_axis == 0 ? d.x : (grid_axis == 1 ? d.y : d.z);
        const float sg = dc > 0.f ? -1.f : 1.f;
        n = f3(grid_axis == 0 ? sg : 0.f, grid_axis == 1 ? sg : 0.f, grid_axis == 2 ? sg : 0.f);
    }
    return n;
}

__device__ __forceinline__ bool inside_bounds(const DevParams& P, F3 p) {
    return p.x >= P.lo[0] && p.x <= P.hi[0] && p.y >= P.lo[1] && p.y <= P.hi[1] &&
           p.z >= P.lo[2] && p.z <= P.hi[2];
}

// Distance from an inside point to the bounds box boundary, less a margin
// for the FP32 rounding of the differences: every point within it of p is
// inside, so a ray may skip the exact test until its chords have used it up.
__device__ __forceinline__ float bounds_free(const DevParams& P, F3 p) {
    const float m = fminf(fminf(fminf(p.x - P.lo[0], P.hi[0] - p.x), fminf(p.y - P.lo[1], P.hi[1] - p.y)),
                          fminf(p.z - P.lo[2], P.hi[2] - p.z));
    return m - 1e-4f - 1e-6f * (fabsf(p.x) + fabsf(p.y) + fabsf(p.z));
}

__device__ __forceinline__ unsigned cell_of(const DevParams& P, F3 p) {
    const int g = P.grid;
    const int ix = min(max((int)floorf((p.x - P.grid_lo[0]) * P.grid_inv[0]), 0), g - 1);
    const int iy = min(max((int)floorf((p.y - P.grid_lo[1]) * P.grid_inv[1]), 0), g - 1);
    const int iz = min(max((int)floorf((p.z - P.grid_lo[2]) * P.grid_inv[2]), 0), g - 1);
    return ((unsigned)iz * g + iy) * g + ix;
}

struct RayResult {
    int status;    // primary: 0 miss 1 hit 2 failed; shadow: 1 lit 0 blocked
    int prim;
    int steps;
    float t;
    F3 point;
    F3 normal;     // NORMAL passes only
};

struct LaneCounters {
    unsigned steps_integrated;
    unsigned bump_evals;
    unsigned lane_slots;       // loop iterations executed by this lane (active or not)
    unsigned jumps;            // integrated steps that were straight jumps (no RK4 / metric work)
};

// March passes.  (A fused lit launch looping over both work kinds through one
// march copy with the pass chosen per work item was measured: ptxas then
// moves every bump loop to the vector datapath — BREV/FLO/LDC instead of
// UBREV/UFLO/LDCU — so the fused launch keeps two loops and two copies.)
enum Pass : int { kPassShade = 0, kPassHits = 1, kPassShadow = 2, kPassFused = 3 };

// ---------------------------------------------------------------------------
// March one warp unit (kernel_impl.hpp:22-94): all 32 lanes step in lockstep
// until every live lane has terminated; retired lanes keep computing (their
// results are locked in), exactly as the reference's retired pack lanes.
// PASS == kPassShadow marches a shadow geodesic (EXTENSION, oracle/rro.c
// shadow_march): lit (1) when it crosses the sphere |x - q| = sqrt(dist2),
// leaves the bounds or runs out of steps; blocked (0) on a nearer hit or a
// metric failure.
template <int KIND, int NB, int PASS, bool MESH>
__device__ __forceinline__ RayResult march_unit_rk23(const DevParams& P, bool live, F3 p, F3 v,
                                                     LaneCounters& cnt, F3 q, float dist2);

template <int KIND, int NB, int SCHEME, int PASS, bool MESH>
__device__ __forceinline__ RayResult march_fixed(const DevParams& P, bool live, F3 p, F3 v,
                                                LaneCounters& cnt, F3 q = F3{0.f, 0.f, 0.f},
                                                float dist2 = 0.f) {
    RayResult res{PASS == kPassShadow ? 1 : 0, -1, 0, 0.f, f3(0.f, 0.f, 0.f), f3(0.f, 0.f, 0.f)};
    bool active = live;
    float cx = 0.f, cy = 0.f, cz = 0.f;       // Kahan compensation of the position sum
    const float h = P.h;
    const float half = 0.5f * h;
    const float sixth = h / 6.f;
    int step = 0;                             // this lane's reference step index
    const float light_d = PASS == kPassShadow ? sqrtf(dist2) : 0.f;
    float mfree = 0.f;                        // mesh free distance budget (EXT meshes)
    float sfree = 0.f;                        // sphere / half-space free distance budget
    // single twist: known at compile time in the NB == 1 diffeo variants (the
    // general fold is then not compiled into the kernel), else checked here
    const bool twist1 = KIND == kDiffeo && (NB == 1 || (P.n_stages == 1 && P.stages[0].kind == kStageTwist));
    for (;;) {
        if (!__any_sync(kFull, active)) break;
        cnt.lane_slots += 1;
        uint32_t um = 0;
        int nj = 0;                           // >= 2: this lane jumps nj straight steps
        if constexpr (KIND == kEuclid) {
            // Gamma = 0 everywhere: every geodesic is the straight line x + j h y,
            // so a lane jumps straight to its bounds exit (or its light's
            // sphere); the chord test finds the hit and its reference step.
            if (P.skip && active) {
                const float speed2 = fmaf(v.x, v.x, fmaf(v.y, v.y, v.z * v.z));
                const float isp = rsqrtf(speed2);
                float te = 3.0e38f;
                if (v.x != 0.f) te = fminf(te, ((v.x > 0.f ? P.hi[0] : P.lo[0]) - p.x) / v.x);
                if (v.y != 0.f) te = fminf(te, ((v.y > 0.f ? P.hi[1] : P.lo[1]) - p.y) / v.y);
                if (v.z != 0.f) te = fminf(te, ((v.z > 0.f ? P.hi[2] : P.lo[2]) - p.z) / v.z);
                float L = te * speed2 * isp;
                if (PASS == kPassShadow) {
                    const F3 r = f3(p.x - q.x, p.y - q.y, p.z - q.z);
                    L = fminf(L, light_d - sqrtf(fmaf(r.x, r.x, fmaf(r.y, r.y, r.z * r.z))));
                }
                const float n = floorf(L * isp / h) - 1.f;
                nj = (int)fminf(fmaxf(n, 0.f), (float)(P.max_steps - step));
                if (nj < 2) nj = 0;
            }
        }
        if constexpr (KIND == kBumps) {
            uint32_t lm = 0;
            unsigned cell = 0;
            if (active) {
                if (P.cull) {
                    cell = cell_of(P, p);
                    lm = __ldg(P.cull_masks + cell);
                } else {
                    lm = P.all_mask;
                }
            }
            // Empty-space skipping: in a cell whose Chebyshev distance to the
            // nearest non-empty cell is k, every point within (k-1) cells is
            // bump-free (6 sigma, dilated by 1.5h), the culled metric is flat
            // and the geodesic is the straight line x + j h y (Gamma = 0), so
            // nj whole steps collapse into one chord.  A jump never crosses the
            // bounds exit or (shadow rays) the light's sphere.
            if (P.skip && active && lm == 0u) {
                const int k = __ldg(P.skip_k + cell);
                if (k >= 2) {
                    const float speed2 = fmaf(v.x, v.x, fmaf(v.y, v.y, v.z * v.z));
                    const float isp = rsqrtf(speed2);
                    float L = (float)(k - 1) * P.cell_min;
                    float te = 3.0e38f;   // parameter distance to the bounds exit along v
                    if (v.x != 0.f) te = fminf(te, ((v.x > 0.f ? P.hi[0] : P.lo[0]) - p.x) / v.x);
                    if (v.y != 0.f) te = fminf(te, ((v.y > 0.f ? P.hi[1] : P.lo[1]) - p.y) / v.y);
                    if (v.z != 0.f) te = fminf(te, ((v.z > 0.f ? P.hi[2] : P.lo[2]) - p.z) / v.z);
                    L = fminf(L, te * speed2 * isp);
                    if (PASS == kPassShadow) {
                        const F3 r = f3(p.x - q.x, p.y - q.y, p.z - q.z);
                        L = fminf(L, light_d - sqrtf(fmaf(r.x, r.x, fmaf(r.y, r.y, r.z * r.z))));
                    }
                    const float n = floorf(L * isp / h) - 1.f;
                    nj = (int)fminf(fmaxf(n, 0.f), (float)(P.max_steps - step));
                    if (nj < 2) nj = 0;
                }
            }
            um = __reduce_or_sync(kFull, nj ? 0u : lm);
            if (active && !nj) cnt.bump_evals += (SCHEME == 0 ? 1u : 4u) * __popc(um);
        }
        float valid = 3.0e38f;
        F3 dp, vn;
        // whole warp jumps: no integration (only Euclidean and bump metrics jump)
        if ((KIND == kEuclid || KIND == kBumps) && __all_sync(kFull, nj != 0 || !active)) {
            dp = f3(0.f, 0.f, 0.f);
            vn = v;
        } else if (SCHEME == 0) {                            // Euler (integrate.hpp:55-61)
            const F3 a = accel<KIND, NB>(P, um, p, v, valid);
            dp = f3(h * v.x, h * v.y, h * v.z);
            vn = f3(fmaf(h, a.x, v.x), fmaf(h, a.y, v.y), fmaf(h, a.z, v.z));
        } else if (KIND == kDiffeo && RR_TWIST_RK4 && twist1) {
            // RK4 of the single twist (integrate.hpp:63-93 with accel_diffeo's
            // closed form): a_z = 0 and a does not depend on z, so z' stays
            // constant, the stage points need no z and dz = h z'.
#if RR_TWIST_XY_PAIRS
            // (x, y) components of one ray as packed pairs: a = vz (vz P +
            // 2 (vy, -vx)) is two FFMA2-class ops on the swizzled velocity
            const F2 P0 = mk2(p.x, p.y), V0 = mk2(v.x, v.y);
            const F2 vz2 = bc2(v.z), two = bc2(2.f);
            const F2 c_half = bc2(half), c_full = bc2(h);
            F2 SX = bc2(0.f), SV = bc2(0.f), Pp = P0, Vp = V0;
#pragma unroll
            for (int st = 0; st < 4; ++st) {
                const F2 swz = mk2(hi2(Vp), -lo2(Vp));                     // (vy, -vx)
                const F2 A = mul2(vz2, fma2(vz2, Pp, mul2(two, swz)));
                if (st == 0 || st == 3) {
                    SX = add2(Vp, SX);
                    SV = add2(A, SV);
                } else {
                    SX = fma2(two, Vp, SX);
                    SV = fma2(two, A, SV);
                }
                const F2 cc = st < 2 ? c_half : c_full;
                Pp = fma2(cc, Vp, P0);
                Vp = fma2(cc, A, V0);
            }
            valid = 1.f;
            const F2 DXY = mul2(bc2(sixth), SX), VXY = fma2(bc2(sixth), SV, V0);
            dp = f3(lo2(DXY), hi2(DXY), h * v.z);
            vn = f3(lo2(VXY), hi2(VXY), v.z);
#else
            float sxx = 0.f, sxy = 0.f, svx = 0.f, svy = 0.f;
            float px = p.x, py = p.y, vx = v.x, vy = v.y;
            const float vz = v.z;
#pragma unroll
            for (int st = 0; st < 4; ++st) {
                const float ax = vz * fmaf(vz, px, 2.f * vy), ay = vz * fmaf(vz, py, -2.f * vx);
                const float wgt = (st == 0 || st == 3) ? 1.f : 2.f;
                sxx = fmaf(wgt, vx, sxx); sxy = fmaf(wgt, vy, sxy);
                svx = fmaf(wgt, ax, svx); svy = fmaf(wgt, ay, svy);
                const float c = st < 2 ? half : h;
                px = fmaf(c, vx, p.x); py = fmaf(c, vy, p.y);
                vx = fmaf(c, ax, v.x); vy = fmaf(c, ay, v.y);
            }
            valid = 1.f;
            dp = f3(sixth * sxx, sixth * sxy, h * vz);
            vn = f3(fmaf(sixth, svx, v.x), fmaf(sixth, svy, v.y), vz);
#endif
        } else {                                             // RK4 (integrate.hpp:63-93)
            F3 sx = f3(0.f, 0.f, 0.f), sv = f3(0.f, 0.f, 0.f);
            F3 ps = p, vs = v;
            auto stage = [&](int st) {
                const F3 a = accel<KIND, NB>(P, um, ps, vs, valid);
                const float wgt = (st == 0 || st == 3) ? 1.f : 2.f;
                sx = f3(fmaf(wgt, vs.x, sx.x), fmaf(wgt, vs.y, sx.y), fmaf(wgt, vs.z, sx.z));
                sv = f3(fmaf(wgt, a.x, sv.x), fmaf(wgt, a.y, sv.y), fmaf(wgt, a.z, sv.z));
                const float c = st < 2 ? half : h;
                ps = f3(fmaf(c, vs.x, p.x), fmaf(c, vs.y, p.y), fmaf(c, vs.z, p.z));
                vs = f3(fmaf(c, a.x, v.x), fmaf(c, a.y, v.y), fmaf(c, a.z, v.z));
            };
            if constexpr (KIND == kDiffeo && RR_DIFFEO_RK4_UNROLL) {   // unrolled stages
#pragma unroll
                for (int st = 0; st < 4; ++st) stage(st);
            } else {
#pragma unroll 1
                for (int st = 0; st < 4; ++st) stage(st);   // one call site: the bump block is inlined once
            }
            dp = f3(sixth * sx.x, sixth * sx.y, sixth * sx.z);
            vn = f3(fmaf(sixth, sv.x, v.x), fmaf(sixth, sv.y, v.y), fmaf(sixth, sv.z, v.z));
        }
        if (nj) {                                            // straight jump of nj steps
            const float hn = h * (float)nj;
            dp = f3(hn * v.x, hn * v.y, hn * v.z);
            vn = v;
            valid = 3.0e38f;
        }
        // Compensated position update: pn = p + dp carrying the rounding error.
        F3 pn;
        {
            const float yx = dp.x - cx, yy = dp.y - cy, yz = dp.z - cz;
            pn = f3(p.x + yx, p.y + yy, p.z + yz);
            cx = (pn.x - p.x) - yx;
            cy = (pn.y - p.y) - yy;
            cz = (pn.z - p.z) - yz;
        }
        if (active) {
            const int nsub = nj ? nj : 1;
            cnt.steps_integrated += 1;
            cnt.jumps += nj ? 1u : 0u;
            float s = 0.f;
            int prim = -1, hid = 0, mrec = 0;
            if (KIND == kDiffeo && !(valid > 1e-14f)) {     // kernel_impl.hpp:54-61
                res.status = PASS == kPassShadow ? 0 : 2;
                res.steps = step;
                active = false;
            } else if (intersect<MESH>(P, p, pn, s, prim, hid, mfree, mrec, sfree)) { // kernel_impl.hpp:63-76
                const F3 pt = f3(fmaf(s, pn.x - p.x, p.x), fmaf(s, pn.y - p.y, p.y),
                                 fmaf(s, pn.z - p.z, p.z));
                const float sj = s * (float)nsub;            // hit position in reference steps
                const int sub = min((int)sj, nsub - 1);
                if constexpr (PASS == kPassShadow) {
                    const F3 r = f3(pt.x - q.x, pt.y - q.y, pt.z - q.z);
                    res.status = (r.x * r.x + r.y * r.y + r.z * r.z) < dist2 ? 0 : 1;
                } else {
                    res.status = 1;
                    res.prim = prim;
                    res.point = pt;
                    res.t = ((float)step + sj) * h;
                    if constexpr (PASS == kPassHits) res.normal = hit_normal(P, hid, s, p, pn, pt, mrec);
                }
                res.steps = step + sub + 1;
                active = false;
            } else if (PASS == kPassShadow &&
                       (pn.x - q.x) * (pn.x - q.x) + (pn.y - q.y) * (pn.y - q.y) +
                               (pn.z - q.z) * (pn.z - q.z) >= dist2) {
                res.status = 1;                              // reached the light's sphere
                res.steps = step + nsub;
                active = false;
            } else if (!inside_bounds(P, pn)) {             // kernel_impl.hpp:77-82
                res.status = PASS == kPassShadow ? 1 : 0;
                res.steps = step + nsub;
                active = false;
            }
            step += nsub;
            if (active && step >= P.max_steps) {             // kernel_impl.hpp:87-91
                res.status = PASS == kPassShadow ? 1 : 0;
                res.steps = P.max_steps;
                active = false;
            }
        }
        p = pn;
        v = vn;
    }
    return res;
}


// ---------------------------------------------------------------------------
// EXTENSION: adaptive Bogacki-Shampine 3(2) march (integrator.scheme "rk23";
// FP64 definition: oracle/rro.c march_one_rk23).  Per-lane step size; FSAL
// (k1 of the next step is k4 of the accepted one); the warp-uniform bump mask
// is taken at the step start and covers every stage point because the
// culling grid is dilated for h_max = 4 h0.  Rejected lanes keep their state.
template <int KIND, int NB, int PASS, bool MESH>
__device__ __forceinline__ RayResult march_unit_rk23(const DevParams& P, bool live, F3 p, F3 v,
                                                     LaneCounters& cnt, F3 q, float dist2) {
    RayResult res{PASS == kPassShadow ? 1 : 0, -1, 0, 0.f, f3(0.f, 0.f, 0.f), f3(0.f, 0.f, 0.f)};
    bool active = live;
    const float h0 = P.h, hmin = h0 / 64.f, hmax = 4.f * h0, tol = P.tol;
    const float light_d = PASS == kPassShadow ? sqrtf(dist2) : 0.f;
    float h = h0, t = 0.f;
    int steps = 0, attempts = 0;
    float mfree = 0.f, sfree = 0.f;
    bool have_k1 = false;
    F3 k1v = f3(0.f, 0.f, 0.f);
    for (;;) {
        if (!__any_sync(kFull, active)) break;
        cnt.lane_slots += 1;
        uint32_t um = 0;
        int nj = 0;                   // >= 2: this lane jumps nj straight steps of h_max
        // Straight jumps: where the (culled) metric is flat the error estimate
        // is ~0, so h sits at h_max and the geodesic is x + j h_max y; a lane
        // at h_max collapses nj such steps into one chord (same rules as the
        // fixed-step march: never past the bounds exit or the light's sphere,
        // bump scenes only inside empty cells of the culling grid).
        float L = -1.f;
        if (P.skip && active && h >= hmax) {
            if constexpr (KIND == kEuclid) L = 3.0e38f;
            if constexpr (KIND == kBumps) {
                if (P.cull) {
                    const unsigned cell = cell_of(P, p);
                    if (__ldg(P.cull_masks + 2u * P.cull_cells + cell) == 0u) {
                        const int k = __ldg(P.skip_k + cell);
                        if (k >= 2) L = (float)(k - 1) * P.cell_min;
                    }
                }
            }
        }
        if (L > 0.f) {
            const float speed2 = fmaf(v.x, v.x, fmaf(v.y, v.y, v.z * v.z));
            const float isp = rsqrtf(speed2);
            float te = 3.0e38f;
            if (v.x != 0.f) te = fminf(te, ((v.x > 0.f ? P.hi[0] : P.lo[0]) - p.x) / v.x);
            if (v.y != 0.f) te = fminf(te, ((v.y > 0.f ? P.hi[1] : P.lo[1]) - p.y) / v.y);
            if (v.z != 0.f) te = fminf(te, ((v.z > 0.f ? P.hi[2] : P.lo[2]) - p.z) / v.z);
            L = fminf(L, te * speed2 * isp);
            if (PASS == kPassShadow) {
                const F3 r = f3(p.x - q.x, p.y - q.y, p.z - q.z);
                L = fminf(L, light_d - sqrtf(fmaf(r.x, r.x, fmaf(r.y, r.y, r.z * r.z))));
            }
            const float n = floorf(L * isp / hmax) - 1.f;
            nj = (int)fminf(fmaxf(n, 0.f), (float)(P.max_steps - steps));
            if (nj < 2) nj = 0;
        }
        if constexpr (KIND == kBumps) {
            uint32_t lm = 0;
            if (active && !nj) {   // the mask level whose dilation covers this lane's h
                const unsigned lvl = h <= h0 ? 0u : (h <= 2.f * h0 ? 1u : 2u);
                lm = P.cull ? __ldg(P.cull_masks + lvl * P.cull_cells + cell_of(P, p)) : P.all_mask;
            }
            um = __reduce_or_sync(kFull, lm);
        }
        float valid = 3.0e38f;
        const bool need_k1 = !__all_sync(kFull, have_k1 || !active);
        if (need_k1) {                         // first step (warp-uniform branch)
            const F3 a = accel<KIND, NB>(P, um, p, v, valid);
            if (!have_k1) k1v = a;
            have_k1 = true;
        }
        const F3 k1x = v;
        F3 k2x, k2v, k3x, k3v, k4x, k4v, xn, vn;
        float e = 0.f;
        if (__all_sync(kFull, nj != 0 || !active)) {   // whole warp jumps: no integration
            k2x = k3x = k4x = v;
            k2v = k3v = k4v = f3(0.f, 0.f, 0.f);
            xn = p;
            vn = v;
        } else {
            // stages k2, k3, k4 through one call site
            F3 ps = f3(fmaf(0.5f * h, k1x.x, p.x), fmaf(0.5f * h, k1x.y, p.y), fmaf(0.5f * h, k1x.z, p.z));
            F3 vs = f3(fmaf(0.5f * h, k1v.x, v.x), fmaf(0.5f * h, k1v.y, v.y), fmaf(0.5f * h, k1v.z, v.z));
#pragma unroll 1
            for (int st = 0; st < 3; ++st) {
                const F3 a = accel<KIND, NB>(P, um, ps, vs, valid);
                if (st == 0) {
                    k2x = vs; k2v = a;
                    ps = f3(fmaf(0.75f * h, k2x.x, p.x), fmaf(0.75f * h, k2x.y, p.y), fmaf(0.75f * h, k2x.z, p.z));
                    vs = f3(fmaf(0.75f * h, k2v.x, v.x), fmaf(0.75f * h, k2v.y, v.y), fmaf(0.75f * h, k2v.z, v.z));
                } else if (st == 1) {
                    k3x = vs; k3v = a;
                    const float c1 = 2.f / 9.f * h, c2 = 1.f / 3.f * h, c3 = 4.f / 9.f * h;
                    xn = f3(fmaf(c1, k1x.x, fmaf(c2, k2x.x, fmaf(c3, k3x.x, p.x))),
                            fmaf(c1, k1x.y, fmaf(c2, k2x.y, fmaf(c3, k3x.y, p.y))),
                            fmaf(c1, k1x.z, fmaf(c2, k2x.z, fmaf(c3, k3x.z, p.z))));
                    vn = f3(fmaf(c1, k1v.x, fmaf(c2, k2v.x, fmaf(c3, k3v.x, v.x))),
                            fmaf(c1, k1v.y, fmaf(c2, k2v.y, fmaf(c3, k3v.y, v.y))),
                            fmaf(c1, k1v.z, fmaf(c2, k2v.z, fmaf(c3, k3v.z, v.z))));
                    ps = xn;
                    vs = vn;
                } else {
                    k4x = vs; k4v = a;
                }
            }
            if constexpr (KIND == kBumps) {
                if (active && !nj) cnt.bump_evals += 3u * __popc(um);
            }
            // embedded error, mixed abs/rel scale
            const float e1 = -5.f / 72.f * h, e2 = 1.f / 12.f * h, e3 = 1.f / 9.f * h, e4 = -1.f / 8.f * h;
            const float y0[6] = {p.x, p.y, p.z, v.x, v.y, v.z};
            const float y1[6] = {xn.x, xn.y, xn.z, vn.x, vn.y, vn.z};
            const float ka[6] = {k1x.x, k1x.y, k1x.z, k1v.x, k1v.y, k1v.z};
            const float kb[6] = {k2x.x, k2x.y, k2x.z, k2v.x, k2v.y, k2v.z};
            const float kc[6] = {k3x.x, k3x.y, k3x.z, k3v.x, k3v.y, k3v.z};
            const float kd[6] = {k4x.x, k4x.y, k4x.z, k4v.x, k4v.y, k4v.z};
#pragma unroll
            for (int i = 0; i < 6; ++i) {
                const float err = fmaf(e1, ka[i], fmaf(e2, kb[i], fmaf(e3, kc[i], e4 * kd[i])));
                const float sc = tol * (1.f + fmaxf(fabsf(y0[i]), fabsf(y1[i])));
                e = fmaxf(e, __fdividef(fabsf(err), sc));
            }
        }
        if (nj) {                                            // straight jump of nj h_max steps
            const float hn = hmax * (float)nj;
            xn = f3(fmaf(hn, v.x, p.x), fmaf(hn, v.y, p.y), fmaf(hn, v.z, p.z));
            vn = v;
            k4v = f3(0.f, 0.f, 0.f);                         // flat (culled) metric at xn
            e = 0.f;
            valid = 3.0e38f;
        }
        const bool accept = e <= 1.f || h <= hmin;
        if (active) {
            const int nsub = nj ? nj : 1;
            const float hstep = nj ? hmax * (float)nj : h;
            cnt.steps_integrated += 1;
            cnt.jumps += nj ? 1u : 0u;
            attempts += nsub;
            float s = 0.f;
            int prim = -1, hid = 0, mrec = 0;
            if (KIND == kDiffeo && !(valid > 1e-14f)) {
                res.status = PASS == kPassShadow ? 0 : 2;
                res.steps = steps;
                active = false;
            } else if (accept) {
                if (intersect<MESH>(P, p, xn, s, prim, hid, mfree, mrec, sfree)) {
                    const F3 pt = f3(fmaf(s, xn.x - p.x, p.x), fmaf(s, xn.y - p.y, p.y),
                                     fmaf(s, xn.z - p.z, p.z));
                    const int sub = min((int)(s * (float)nsub), nsub - 1);
                    if constexpr (PASS == kPassShadow) {
                        const F3 r = f3(pt.x - q.x, pt.y - q.y, pt.z - q.z);
                        res.status = (r.x * r.x + r.y * r.y + r.z * r.z) < dist2 ? 0 : 1;
                    } else {
                        res.status = 1;
                        res.prim = prim;
                        res.point = pt;
                        res.t = fmaf(s, hstep, t);
                        if constexpr (PASS == kPassHits) res.normal = hit_normal(P, hid, s, p, xn, pt, mrec);
                    }
                    res.steps = steps + sub + 1;
                    active = false;
                } else {
                    steps += nsub;
                    const bool crossed = PASS == kPassShadow &&
                        (xn.x - q.x) * (xn.x - q.x) + (xn.y - q.y) * (xn.y - q.y) +
                            (xn.z - q.z) * (xn.z - q.z) >= dist2;
                    if (crossed || !inside_bounds(P, xn)) {
                        res.status = PASS == kPassShadow ? 1 : 0;
                        res.steps = steps;
                        active = false;
                    } else {
                        t += hstep;
                        p = xn;
                        v = vn;
                        k1v = k4v;
                    }
                }
            }
            if (active) {
                const float fac = e > 0.f ? fminf(5.f, fmaxf(0.2f, 0.9f * ex2(-__log2f(e) / 3.f))) : 5.f;
                h = fminf(hmax, fmaxf(hmin, h * fac));
                if (steps >= P.max_steps || attempts >= 16 * P.max_steps) {
                    res.status = PASS == kPassShadow ? 1 : 0;
                    res.steps = steps;
                    active = false;
                }
            }
        }
    }
    return res;
}

template <int KIND, int NB, int SCHEME, int PASS, bool MESH>
__device__ __forceinline__ RayResult march_unit(const DevParams& P, bool live, F3 p, F3 v,
                                                LaneCounters& cnt, F3 q = F3{0.f, 0.f, 0.f},
                                                float dist2 = 0.f) {
    if constexpr (SCHEME == 2) return march_unit_rk23<KIND, NB, PASS, MESH>(P, live, p, v, cnt, q, dist2);
    else return march_fixed<KIND, NB, SCHEME, PASS, MESH>(P, live, p, v, cnt, q, dist2);
}

// g at x (metric.cpp:12-15 / :40-42), for the shadow ray's unit g-speed.
__device__ void metric_at(const DevParams& P, F3 x, float g[6], bool& ok) {
    float gx = 0.f, gy = 0.f, gz = 0.f;   // grad f (graph) ; J (diffeo) below
    ok = true;
    g[0] = g[3] = g[5] = 1.f;
    g[1] = g[2] = g[4] = 0.f;
    if (P.kind == kBumps || P.kind == kGraphGeneral) {
        for (int j = 0; j < (P.kind == kBumps ? P.nb_slot : P.n_bumps); ++j) {
            const DevBump& b = P.bumps[j];
            const float dx = x.x - b.cx, dy = x.y - b.cy, dz = x.z - b.cz;
            const float v = ex2(fmaf(dx * b.kx, dx, fmaf(dy * b.ky, dy, fmaf(dz * b.kz, dz, b.la)))) * b.sgn;
            gx = fmaf(-v * kBeta, dx * b.kx, gx);
            gy = fmaf(-v * kBeta, dy * b.ky, gy);
            gz = fmaf(-v * kBeta, dz * b.kz, gz);
        }
        float xp[5], yp[5], zp[5];
        xp[0] = yp[0] = zp[0] = 1.f;
        for (int k = 1; k < 5; ++k) {
            xp[k] = xp[k - 1] * x.x;
            yp[k] = yp[k - 1] * x.y;
            zp[k] = zp[k - 1] * x.z;
        }
        for (int i = 0; i < P.n_poly; ++i) {
            const DevPoly& t = P.poly[i];
            if (t.a > 0) gx = fmaf(t.coef * t.a, xp[t.a - 1] * yp[t.b] * zp[t.c], gx);
            if (t.b > 0) gy = fmaf(t.coef * t.b, xp[t.a] * yp[t.b - 1] * zp[t.c], gy);
            if (t.c > 0) gz = fmaf(t.coef * t.c, xp[t.a] * yp[t.b] * zp[t.c - 1], gz);
        }
        g[0] += gx * gx; g[1] = gx * gy; g[2] = gx * gz;
        g[3] += gy * gy; g[4] = gy * gz; g[5] += gz * gz;
    } else if (P.kind == kDiffeo) {
        float J[9] = {1.f, 0.f, 0.f, 0.f, 1.f, 0.f, 0.f, 0.f, 1.f};
        float x0 = x.x, x1 = x.y, x2 = x.z;
        for (int s = 0; s < P.n_stages; ++s) {
            const DevStage& st = P.stages[s];
            float Js[9], n0, n1, n2;
            if (st.kind == kStageAffine) {
                for (int k = 0; k < 9; ++k) Js[k] = st.v[k];
                n0 = st.v[0] * x0 + st.v[1] * x1 + st.v[2] * x2 + st.v[9];
                n1 = st.v[3] * x0 + st.v[4] * x1 + st.v[5] * x2 + st.v[10];
                n2 = st.v[6] * x0 + st.v[7] * x1 + st.v[8] * x2 + st.v[11];
            } else if (st.kind == kStageTwist) {
                float sn, cs;
                sincosf(x2, &sn, &cs);
                Js[0] = cs; Js[1] = -sn; Js[2] = -(x0 * sn) - x1 * cs;
                Js[3] = sn; Js[4] = cs; Js[5] = x0 * cs - x1 * sn;
                Js[6] = 0.f; Js[7] = 0.f; Js[8] = 1.f;
                n0 = x0 * cs - x1 * sn;
                n1 = x0 * sn + x1 * cs;
                n2 = x2;
            } else if (st.kind == kStageBend) {
                const float k = st.v[0], c = st.v[1];
                float sn, cs;
                __sincosf(k * x0, &sn, &cs);
                const float yc = x1 - c;
                Js[0] = -k * cs * yc; Js[1] = -sn; Js[2] = 0.f;
                Js[3] = -k * sn * yc; Js[4] = cs; Js[5] = 0.f;
                Js[6] = 0.f; Js[7] = 0.f; Js[8] = 1.f;
                n0 = -sn * yc;
                n1 = fmaf(cs, yc, c);
                n2 = x2;
            } else {
                const float* b = st.v;
                const float ux = (x0 - b[0]) * b[3], uy = (x1 - b[1]) * b[4], uz = (x2 - b[2]) * b[5];
                const float e = b[6] * __expf(-0.5f * (ux * ux + uy * uy + uz * uz));
                const float fg[3] = {-e * ux * b[3], -e * uy * b[4], -e * uz * b[5]};
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j) Js[3 * i + j] = (i == j ? 1.f : 0.f) + b[7 + i] * fg[j];
                n0 = fmaf(e, b[7], x0);
                n1 = fmaf(e, b[8], x1);
                n2 = fmaf(e, b[9], x2);
            }
            float R[9];
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j)
                    R[3 * i + j] = Js[3 * i] * J[j] + Js[3 * i + 1] * J[3 + j] + Js[3 * i + 2] * J[6 + j];
            for (int k = 0; k < 9; ++k) J[k] = R[k];
            x0 = n0; x1 = n1; x2 = n2;
        }
        const float d = J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) +
                        J[2] * (J[3] * J[7] - J[4] * J[6]);
        ok = fabsf(d) > 1e-14f;
        g[0] = J[0] * J[0] + J[3] * J[3] + J[6] * J[6];
        g[1] = J[0] * J[1] + J[3] * J[4] + J[6] * J[7];
        g[2] = J[0] * J[2] + J[3] * J[5] + J[6] * J[8];
        g[3] = J[1] * J[1] + J[4] * J[4] + J[7] * J[7];
        g[4] = J[1] * J[2] + J[4] * J[5] + J[7] * J[8];
        g[5] = J[2] * J[2] + J[5] * J[5] + J[8] * J[8];
    }
}

// Pseudo-colour + fog (render.cpp:14-25) packed r | g << 8 | b << 16;
// failures magenta (render.cpp:39).  `light` scales the colour (EXTENSION lit
// shading; 1 = reference shading).
__device__ __forceinline__ uint32_t shade_rgb(const DevParams& P, int status, float t, F3 point,
                                              float light = 1.f) {
    if (status == 2) return 0xff00ffu;
    if (status != 1) return 0u;
    const float atten = expf(-P.fog * t);
    const float pv[3] = {point.x, point.y, point.z};
    uint32_t c = 0u;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float frac = pv[k] - floorf(pv[k]);
        // lround (half away from zero) for the non-negative argument (see shade)
        const float x = 255.f * (frac * atten * light);
        const float tr = truncf(x);
        int v = (int)tr + ((x - tr) >= 0.5f ? 1 : 0);
        v = v < 0 ? 0 : (v > 255 ? 255 : v);
        c |= (uint32_t)v << (8 * k);
    }
    return c;
}

__device__ __forceinline__ void shade(const DevParams& P, const RayResult& r, uint8_t* rgb,
                                      float light = 1.f) {
    if (r.status == 2) {
        rgb[0] = 255; rgb[1] = 0; rgb[2] = 255;
        return;
    }
    if (r.status != 1) {
        rgb[0] = rgb[1] = rgb[2] = 0;
        return;
    }
    const float atten = expf(-P.fog * r.t);
    const float pv[3] = {r.point.x, r.point.y, r.point.z};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float frac = pv[k] - floorf(pv[k]);
        // lround (half away from zero) for the non-negative argument, without
        // the 64-bit conversion code of lroundf: trunc + exact fraction test
        const float x = 255.f * (frac * atten * light);
        const float tr = truncf(x);
        int v = (int)tr + ((x - tr) >= 0.5f ? 1 : 0);
        v = v < 0 ? 0 : (v > 255 ? 255 : v);
        rgb[k] = (uint8_t)v;
    }
}

// Primary ray of pixel (px, py) (camera.cpp:22-29), computed in FP64.
__device__ __forceinline__ void raygen(const DevCamera& c, int px, int py, int w, int h, F3& pos,
                                       F3& dir) {
    const double sx = (2.0 * (px + 0.5) / w - 1.0) * c.tan_half * c.aspect;
    const double sy = (1.0 - 2.0 * (py + 0.5) / h) * c.tan_half;
    const double dx = c.f0[0] + sx * c.f2[0] + sy * c.f1[0];
    const double dy = c.f0[1] + sx * c.f2[1] + sy * c.f1[1];
    const double dz = c.f0[2] + sx * c.f2[2] + sy * c.f1[2];
    const double n2 = c.g[0] * dx * dx + c.g[3] * dy * dy + c.g[5] * dz * dz +
                      2.0 * (c.g[1] * dx * dy + c.g[2] * dx * dz + c.g[4] * dy * dz);
    const double inv = 1.0 / sqrt(n2);
    pos = f3((float)c.pos[0], (float)c.pos[1], (float)c.pos[2]);
    dir = f3((float)(dx * inv), (float)(dy * inv), (float)(dz * inv));
}

// ---------------------------------------------------------------------------
// Ray-pair march (Gaussian-bump metric, fixed-step RK4, mesh-free scenes):
// march_fixed for two rays per thread.  The integrator and the metric run
// packed (F2 / P3); the culling lookup, the chord test and the termination
// bookkeeping run per ray on the unpacked halves with exactly march_fixed's
// rules (kernel_impl.hpp:22-94).  The warp-uniform bump mask is the OR over
// the 64 rays of the unit.
template <int PASS>
__device__ __forceinline__ int jump_steps(const DevParams& P, F3 p, F3 v, int k, int step, F3 q,
                                          float light_d, bool shadow = PASS == kPassShadow,
                                          float inv_step = 0.f) {
    const float speed2 = fmaf(v.x, v.x, fmaf(v.y, v.y, v.z * v.z));
    const float isp = rsqrtf(speed2);
    float L = (float)(k - 1) * P.cell_min;
    float te = 3.0e38f;   // parameter distance to the bounds exit along v
    if (v.x != 0.f) te = fminf(te, __fdividef((v.x > 0.f ? P.hi[0] : P.lo[0]) - p.x, v.x));
    if (v.y != 0.f) te = fminf(te, __fdividef((v.y > 0.f ? P.hi[1] : P.lo[1]) - p.y, v.y));
    if (v.z != 0.f) te = fminf(te, __fdividef((v.z > 0.f ? P.hi[2] : P.lo[2]) - p.z, v.z));
    L = fminf(L, te * speed2 * isp);
    if (shadow) {
        const F3 r = f3(p.x - q.x, p.y - q.y, p.z - q.z);
        L = fminf(L, light_d - sqrtf(fmaf(r.x, r.x, fmaf(r.y, r.y, r.z * r.z))));
    }
    // fast division: the -1 step margin covers it
    const float n = floorf(L * isp * (inv_step > 0.f ? inv_step : P.inv_h)) - 1.f;
    const int nj = (int)fminf(fmaxf(n, 0.f), (float)(P.max_steps - step));
    return nj < 2 ? 0 : nj;
}

template <int PASS>
__device__ __forceinline__ void emit_primary(const DevParams& P, const DevLaunch& L, unsigned unit,
                                             int r, const RayResult& res);

// Per-warp shared-memory staging of a ray-pair unit's primary results: a ray
// that terminates parks {t, point} and {status | (prim+1) << 8, steps} here
// (two shared stores) instead of holding them in registers for the rest of
// the unit's march; the unit's epilogue shades all 64 pixels at once, writes
// the optional PixelOutcome records, and stores the 16x4-pixel RGB block
// with 16-byte stores (rgb: 4 rows x 48 bytes).
struct PairStage {
    float4 tp[2 * kUnit];     // t, point.x, point.y, point.z
    int2 sp[2 * kUnit];       // status | (prim + 1) << 8, steps
    uint32_t rgb[48];         // 4 rows x 48 bytes of the 16x4 pixel block
    float4* chord;            // kPassHits (RR_X2_HITS_STAGED): 4 x 32 float4 per ray pair unit —
                              // [r][lane] = (chord start, s), [2 + r][lane] = (chord end,
                              // hid | mrec << 12) — so the hit normal and the 32-B hit
                              // record are produced after the march, not inside its loop
};

// render::PixelOutcome (kernel.hpp:33-39, 48 B) from FP32 results: prim -1,
// point 0 and t 0 unless hit, exactly as march_kernel's batch mode.
__device__ __forceinline__ void write_outcome(uint8_t* base, unsigned long long idx, int status,
                                              int prim, F3 pt, float t, int steps,
                                              unsigned long long cap) {
    RR_CHECK(idx < cap, "outcome index");
    const bool hit = status == 1;
    const double x = hit ? (double)pt.x : 0.0, y = hit ? (double)pt.y : 0.0;
    const double z = hit ? (double)pt.z : 0.0, tt = hit ? (double)t : 0.0;
    int4* o = reinterpret_cast<int4*>(base + 48ull * idx);
    o[0] = make_int4(status & 0xff, hit ? prim : -1, __double2loint(x), __double2hiint(x));
    o[1] = make_int4(__double2loint(y), __double2hiint(y), __double2loint(z), __double2hiint(z));
    o[2] = make_int4(__double2loint(tt), __double2hiint(tt), steps, 0);
}

// Marches a ray pair.  Every ray's output is emitted when it terminates:
// kPassShade parks it in the warp's PairStage, kPassHits writes the hit
// record (emit_primary), kPassShadow returns per-ray status and
// reference-equivalent step counts.  Primary passes accumulate the unit's
// reference steps / failures into `us` (no per-ray outputs stay live in
// registers through the march).
struct UnitStats {
    LaneCounters cnt;
    unsigned ref_steps, errs, shadow_steps, nrays;
};

// Packed RK4 of the single twist (march_fixed's closed form, two rays per
// thread): a_z = 0 and a does not depend on z, so z' stays constant, the
// stage points need no z and dz = h z' (integrate.hpp:63-93).
__device__ __forceinline__ void twist_rk4_x2(const P3& p, const P3& v, F2 half, F2 full, F2 sixth,
                                             P3& dp, P3& vn) {
    const F2 two = bc2(2.f), mtwo = bc2(-2.f);
    F2 sxx = bc2(0.f), sxy = bc2(0.f), svx = bc2(0.f), svy = bc2(0.f);
    F2 px = p.x, py = p.y, vx = v.x, vy = v.y;
    const F2 vz = v.z;
#pragma unroll
    for (int st = 0; st < 4; ++st) {
        const F2 ax = mul2(vz, fma2(vz, px, mul2(two, vy)));
        const F2 ay = mul2(vz, fma2(vz, py, mul2(mtwo, vx)));
        if (st == 0 || st == 3) {
            sxx = add2(vx, sxx); sxy = add2(vy, sxy);
            svx = add2(ax, svx); svy = add2(ay, svy);
        } else {
            sxx = fma2(two, vx, sxx); sxy = fma2(two, vy, sxy);
            svx = fma2(two, ax, svx); svy = fma2(two, ay, svy);
        }
        const F2 cc = st < 2 ? half : full;
        px = fma2(cc, vx, p.x); py = fma2(cc, vy, p.y);
        vx = fma2(cc, ax, v.x); vy = fma2(cc, ay, v.y);
    }
    dp = P3{mul2(sixth, sxx), mul2(sixth, sxy), mul2(full, vz)};
    vn = P3{fma2(sixth, svx, v.x), fma2(sixth, svy, v.y), vz};
}

// Mesh part of intersect() for one ray (MESH pair marches): the chord
// [a, a + d] against every mesh, then the free ball at its end.  The pair
// kernel has one call site (the compacted test loop), so the traversals are
// inlined there (RR_MESH_INLINE_PAIRS): a call would save and restore the
// live state of both rays around it.
#ifndef RR_MESH_INLINE_PAIRS
#define RR_MESH_INLINE_PAIRS 1
#endif
__device__ __forceinline__ void mesh_part(const DevParams& P, F3 a, F3 d, float len, bool& have,
                                          float& s_best, int& prim, int& hid, int& mrec, float& mfree) {
    for (int i = 0; i < P.n_meshes; ++i) {
        int rec = 0;
        float s = 0.f;
        const bool h = RR_MESH_INLINE_PAIRS ? mesh_chord_impl(P.meshes[i], a, d, s, rec)
                                            : mesh_chord(P.meshes[i], a, d, s, rec);
        if (consider(h, s, P.meshes[i].index, (kPrimMesh << 8) | i, have, s_best, prim, hid)) mrec = rec;
    }
    const F3 b = f3(a.x + d.x, a.y + d.y, a.z + d.z);
    float fr = 3.0e38f;
    for (int i = 0; i < P.n_meshes; ++i)
        fr = fminf(fr, RR_MESH_INLINE_PAIRS ? mesh_free_impl(P.meshes[i], b, RR_MESH_FREE_CAP)
                                            : mesh_free(P.meshes[i], b, RR_MESH_FREE_CAP));
    mfree = fr;
}

// EXTENSION: the adaptive Bogacki-Shampine 3(2) march (march_unit_rk23,
// oracle/rro.c rk23_core) for a ray pair: per-ray step size h, FSAL k1, the
// three stage evaluations packed (FFMA2) with per-ray coefficients, the
// embedded error norm and the step-size control per ray; bump mask from the
// culling level that covers each ray's h, OR-reduced over the warp's 64 rays;
// rays at h_max in empty cells take straight jumps of h_max steps.  Output
// rules exactly as march_pair.
template <int NB, int PASS>
__device__ __forceinline__ void march_pair_rk23(const DevParams& P, bool live0, bool live1, P3 p, P3 v,
                                                UnitStats& us, const DevLaunch& L, unsigned unit,
                                                int (&status)[2], int (&steps)[2], PairStage* stg,
                                                F3 q0, F3 q1, float d20, float d21) {
    constexpr bool kShadow = PASS == kPassShadow;
    constexpr bool kHits = PASS == kPassHits;
    LaneCounters& cnt = us.cnt;
    const int lane = threadIdx.x & 31;
    status[0] = status[1] = kShadow ? 1 : 0;
    steps[0] = steps[1] = 0;
    bool act[2] = {live0, live1};
    const F3 qq[2] = {q0, q1};
    const float dd[2] = {d20, d21};
    float light_d[2] = {0.f, 0.f};
    if (kShadow) {
        light_d[0] = sqrtf(d20);
        light_d[1] = sqrtf(d21);
    }
    const float h0 = P.h, hmin = h0 / 64.f, hmax = 4.f * h0, tol = P.tol;
    const float inv_hmax = 0.25f * P.inv_h;
    float hh[2] = {h0, h0}, tt[2] = {0.f, 0.f};
    int stp[2] = {0, 0}, att[2] = {0, 0};
    bool have_k1[2] = {false, false};
    P3 k1v{bc2(0.f), bc2(0.f), bc2(0.f)};
    float sfree[2] = {0.f, 0.f};
#if RR_RK23_K1_PRELOOP
    // k1 = a(x0, y0) of every ray before the loop (FSAL afterwards), so the
    // loop body carries three inlined bump blocks instead of four.  The first
    // attempt never jumps (h = h0 < h_max), so this is the mask the loop's
    // first attempt would use: level 0 at each live ray's cell.
    if (__any_sync(kFull, act[0] || act[1])) {
        uint32_t l0 = 0u;
#pragma unroll
        for (int r = 0; r < 2; ++r)
            if (act[r]) l0 |= P.cull ? __ldg(P.cull_masks + cell_of(P, ray_of(p, r))) : P.all_mask;
        const uint32_t um0 = __reduce_or_sync(kFull, l0);
        k1v = accel_bumps_x2<NB, RR_X2_SCALAR_CONSTS_RK23>(P, um0, p, v);   // (not in bump_evals, as before)
    }
    have_k1[0] = have_k1[1] = true;
#endif
    for (;;) {
        if (!__any_sync(kFull, act[0] || act[1])) break;
        cnt.lane_slots += 2;
        int nj[2] = {0, 0};
        uint32_t lmo = 0u;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            if (!act[r]) continue;
            unsigned cell = 0;
            if (P.cull) cell = cell_of(P, ray_of(p, r));
            // straight jumps: a ray at h_max in a cell empty at the widest
            // level (dilated for 4 h0) moves x + j h_max y (rk23 in flat space)
            if (P.skip && P.cull && hh[r] >= hmax && __ldg(P.cull_masks + 2u * P.cull_cells + cell) == 0u) {
                const int k = __ldg(P.skip_k + cell);
                if (k >= 2)
                    nj[r] = jump_steps<PASS>(P, ray_of(p, r), ray_of(v, r), k, stp[r], qq[r], light_d[r],
                                             kShadow, inv_hmax);
            }
            if (!nj[r]) {   // the mask level whose dilation covers this ray's h
                const unsigned lvl = hh[r] <= h0 ? 0u : (hh[r] <= 2.f * h0 ? 1u : 2u);
                lmo |= P.cull ? __ldg(P.cull_masks + lvl * P.cull_cells + cell) : P.all_mask;
            }
        }
        const uint32_t um = __reduce_or_sync(kFull, lmo);
        // first step of a ray: k1 = a(x, y) (FSAL afterwards)
        if (!RR_RK23_K1_PRELOOP && !__all_sync(kFull, (have_k1[0] || !act[0]) && (have_k1[1] || !act[1]))) {
            const P3 a = accel_bumps_x2<NB, RR_X2_SCALAR_CONSTS_RK23>(P, um, p, v);
            k1v = P3{sel2(have_k1[0], have_k1[1], k1v.x, a.x), sel2(have_k1[0], have_k1[1], k1v.y, a.y),
                     sel2(have_k1[0], have_k1[1], k1v.z, a.z)};
            have_k1[0] = have_k1[1] = true;
        }
        P3 xn = p, vn = v, k4v{bc2(0.f), bc2(0.f), bc2(0.f)};
        float e[2] = {0.f, 0.f};
        const bool jw0 = nj[0] != 0 || !act[0], jw1 = nj[1] != 0 || !act[1];
        if (!__all_sync(kFull, jw0 && jw1)) {
#pragma unroll
            for (int r = 0; r < 2; ++r)
                if (act[r] && !nj[r]) cnt.bump_evals += 3u * __popc(um);
            const F2 H = mk2(hh[0], hh[1]);
            const F2 c05 = mul2(bc2(0.5f), H), c075 = mul2(bc2(0.75f), H);
            // stages k2, k3, k4 (march_unit_rk23 order of operations)
            P3 ps{fma2(c05, v.x, p.x), fma2(c05, v.y, p.y), fma2(c05, v.z, p.z)};
            P3 vs{fma2(c05, k1v.x, v.x), fma2(c05, k1v.y, v.y), fma2(c05, k1v.z, v.z)};
            const P3 k2x = vs;
            const P3 k2v = accel_bumps_x2<NB, RR_X2_SCALAR_CONSTS_RK23>(P, um, ps, vs);
            ps = P3{fma2(c075, k2x.x, p.x), fma2(c075, k2x.y, p.y), fma2(c075, k2x.z, p.z)};
            vs = P3{fma2(c075, k2v.x, v.x), fma2(c075, k2v.y, v.y), fma2(c075, k2v.z, v.z)};
            const P3 k3x = vs;
            const P3 k3v = accel_bumps_x2<NB, RR_X2_SCALAR_CONSTS_RK23>(P, um, ps, vs);
            const F2 c1 = mul2(bc2(2.f / 9.f), H), c2 = mul2(bc2(1.f / 3.f), H), c3 = mul2(bc2(4.f / 9.f), H);
            xn = P3{fma2(c1, v.x, fma2(c2, k2x.x, fma2(c3, k3x.x, p.x))),
                    fma2(c1, v.y, fma2(c2, k2x.y, fma2(c3, k3x.y, p.y))),
                    fma2(c1, v.z, fma2(c2, k2x.z, fma2(c3, k3x.z, p.z)))};
            vn = P3{fma2(c1, k1v.x, fma2(c2, k2v.x, fma2(c3, k3v.x, v.x))),
                    fma2(c1, k1v.y, fma2(c2, k2v.y, fma2(c3, k3v.y, v.y))),
                    fma2(c1, k1v.z, fma2(c2, k2v.z, fma2(c3, k3v.z, v.z)))};
            const P3 k4x = vn;
            k4v = accel_bumps_x2<NB, RR_X2_SCALAR_CONSTS_RK23>(P, um, xn, vn);
            // embedded error, mixed abs/rel scale, per ray
            const F2 e1 = mul2(bc2(-5.f / 72.f), H), e2 = mul2(bc2(1.f / 12.f), H);
            const F2 e3 = mul2(bc2(1.f / 9.f), H), e4 = mul2(bc2(-1.f / 8.f), H);
            const F2 ka[6] = {v.x, v.y, v.z, k1v.x, k1v.y, k1v.z};
            const F2 kb[6] = {k2x.x, k2x.y, k2x.z, k2v.x, k2v.y, k2v.z};
            const F2 kc[6] = {k3x.x, k3x.y, k3x.z, k3v.x, k3v.y, k3v.z};
            const F2 kd[6] = {k4x.x, k4x.y, k4x.z, k4v.x, k4v.y, k4v.z};
            const F2 y0[6] = {p.x, p.y, p.z, v.x, v.y, v.z};
            const F2 y1[6] = {xn.x, xn.y, xn.z, vn.x, vn.y, vn.z};
#pragma unroll
            for (int i = 0; i < 6; ++i) {
                const F2 err = fma2(e1, ka[i], fma2(e2, kb[i], fma2(e3, kc[i], mul2(e4, kd[i]))));
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const float sc = tol * (1.f + fmaxf(fabsf(get2(y0[i], r)), fabsf(get2(y1[i], r))));
                    e[r] = fmaxf(e[r], __fdividef(fabsf(get2(err, r)), sc));
                }
            }
        }
        if (nj[0] | nj[1]) {                                 // straight jumps of nj h_max steps
            const F2 hn = mk2(hmax * (float)nj[0], hmax * (float)nj[1]);
            const bool j0 = nj[0] != 0, j1 = nj[1] != 0;
            const P3 xj{fma2(hn, v.x, p.x), fma2(hn, v.y, p.y), fma2(hn, v.z, p.z)};
            xn = P3{sel2(j0, j1, xj.x, xn.x), sel2(j0, j1, xj.y, xn.y), sel2(j0, j1, xj.z, xn.z)};
            vn = P3{sel2(j0, j1, v.x, vn.x), sel2(j0, j1, v.y, vn.y), sel2(j0, j1, v.z, vn.z)};
            const F2 z = bc2(0.f);
            k4v = P3{sel2(j0, j1, z, k4v.x), sel2(j0, j1, z, k4v.y), sel2(j0, j1, z, k4v.z)};
            if (j0) e[0] = 0.f;
            if (j1) e[1] = 0.f;
        }
        bool upd[2] = {false, false};   // accepted, still marching: the state moves to (xn, vn)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            if (!act[r]) continue;
            const bool accept = e[r] <= 1.f || hh[r] <= hmin;
            const int nsub = nj[r] ? nj[r] : 1;
            const float hstep = nj[r] ? hmax * (float)nj[r] : hh[r];
            cnt.steps_integrated += 1;
            cnt.jumps += nj[r] ? 1u : 0u;
            att[r] += nsub;
            if (accept) {
                const F3 a = ray_of(p, r), b = ray_of(xn, r);
                float s = 0.f, md = 0.f;
                int prim = -1, hid = 0, mr = 0;
                if (intersect<false>(P, a, b, s, prim, hid, md, mr, sfree[r])) {
                    const F3 pt = f3(fmaf(s, b.x - a.x, a.x), fmaf(s, b.y - a.y, a.y), fmaf(s, b.z - a.z, a.z));
                    const int sub = min((int)(s * (float)nsub), nsub - 1);
                    if constexpr (kShadow) {
                        const F3 rr = f3(pt.x - qq[r].x, pt.y - qq[r].y, pt.z - qq[r].z);
                        status[r] = (rr.x * rr.x + rr.y * rr.y + rr.z * rr.z) < dd[r] ? 0 : 1;
                        steps[r] = stp[r] + sub + 1;
                    } else {
                        const float th = fmaf(s, hstep, tt[r]);
                        const int nst = stp[r] + sub + 1;
                        if constexpr (kHits && !RR_X2_HITS_STAGED) {
                            RayResult res{1, prim, nst, th, pt, f3(0.f, 0.f, 0.f)};
                            res.normal = hit_normal(P, hid, s, a, b, pt, 0);
                            emit_primary<kPassHits>(P, L, unit, r, res);
                        } else {
                            if constexpr (kHits) {
                                stg->chord[r * kUnit + lane] = make_float4(a.x, a.y, a.z, s);
                                stg->chord[(2 + r) * kUnit + lane] =
                                    make_float4(b.x, b.y, b.z, __int_as_float(hid));
                            }
                            stg->tp[r * kUnit + lane] = make_float4(th, pt.x, pt.y, pt.z);
                            stg->sp[r * kUnit + lane] = make_int2(1 | ((prim + 1) << 8), nst);
                        }
                        us.ref_steps += (unsigned)nst;
                    }
                    act[r] = false;
                } else {
                    stp[r] += nsub;
                    const bool crossed = kShadow && (b.x - qq[r].x) * (b.x - qq[r].x) +
                                                            (b.y - qq[r].y) * (b.y - qq[r].y) +
                                                            (b.z - qq[r].z) * (b.z - qq[r].z) >= dd[r];
                    if (crossed || !inside_bounds(P, b)) {
                        act[r] = false;
                        if constexpr (kShadow) {
                            status[r] = 1;
                            steps[r] = stp[r];
                        } else {
                            if constexpr (kHits && !RR_X2_HITS_STAGED) {
                                RayResult res{0, -1, stp[r], 0.f, f3(0.f, 0.f, 0.f), f3(0.f, 0.f, 0.f)};
                                emit_primary<kPassHits>(P, L, unit, r, res);
                            } else {
                                stg->tp[r * kUnit + lane] = make_float4(0.f, 0.f, 0.f, 0.f);
                                stg->sp[r * kUnit + lane] = make_int2(0, stp[r]);
                            }
                            us.ref_steps += (unsigned)stp[r];
                        }
                    } else {
                        tt[r] += hstep;
                        upd[r] = true;
                    }
                }
            }
            if (act[r]) {
                const float fac = e[r] > 0.f ? fminf(5.f, fmaxf(0.2f, 0.9f * ex2(-__log2f(e[r]) / 3.f))) : 5.f;
                hh[r] = fminf(hmax, fmaxf(hmin, hh[r] * fac));
                if (stp[r] >= P.max_steps || att[r] >= 16 * P.max_steps) {
                    act[r] = false;
                    if constexpr (kShadow) {
                        status[r] = 1;
                        steps[r] = stp[r];
                    } else {
                        if constexpr (kHits && !RR_X2_HITS_STAGED) {
                            RayResult res{0, -1, stp[r], 0.f, f3(0.f, 0.f, 0.f), f3(0.f, 0.f, 0.f)};
                            emit_primary<kPassHits>(P, L, unit, r, res);
                        } else {
                            stg->tp[r * kUnit + lane] = make_float4(0.f, 0.f, 0.f, 0.f);
                            stg->sp[r * kUnit + lane] = make_int2(0, stp[r]);
                        }
                        us.ref_steps += (unsigned)stp[r];
                    }
                }
            }
        }
        p = P3{sel2(upd[0], upd[1], xn.x, p.x), sel2(upd[0], upd[1], xn.y, p.y), sel2(upd[0], upd[1], xn.z, p.z)};
        v = P3{sel2(upd[0], upd[1], vn.x, v.x), sel2(upd[0], upd[1], vn.y, v.y), sel2(upd[0], upd[1], vn.z, v.z)};
        k1v = P3{sel2(upd[0], upd[1], k4v.x, k1v.x), sel2(upd[0], upd[1], k4v.y, k1v.y),
                 sel2(upd[0], upd[1], k4v.z, k1v.z)};
    }
}

template <int KIND, int NB, int PASS, bool MESH>
__device__ __forceinline__ void march_pair(const DevParams& P, bool live0, bool live1, P3 p, P3 v,
                                           UnitStats& us, const DevLaunch& L, unsigned unit,
                                           int (&status)[2], int (&steps)[2], PairStage* stg,
                                           F3 q0 = F3{0.f, 0.f, 0.f},
                                           F3 q1 = F3{0.f, 0.f, 0.f}, float d20 = 0.f, float d21 = 0.f) {
    static_assert(KIND == kBumps || KIND == kDiffeo || KIND == kBumpsRk23 || KIND == kDiffeoChain,
                  "ray pairs: Gaussian bumps (RK4 / rk23), the single twist or diffeo chains");
    if constexpr (KIND == kBumpsRk23) {
        march_pair_rk23<NB, PASS>(P, live0, live1, p, v, us, L, unit, status, steps, stg, q0, q1, d20, d21);
        return;
    }
    constexpr bool kShadow = PASS == kPassShadow;
    constexpr bool kHits = PASS == kPassHits;
    LaneCounters& cnt = us.cnt;
    const int lane = threadIdx.x & 31;
    status[0] = status[1] = kShadow ? 1 : 0;
    steps[0] = steps[1] = 0;
    bool act[2] = {live0, live1};
    int step[2] = {0, 0};
    const F3 qq[2] = {q0, q1};
    const float dd[2] = {d20, d21};
    float light_d[2] = {0.f, 0.f};
    if (kShadow) {
        light_d[0] = sqrtf(d20);
        light_d[1] = sqrtf(d21);
    }
    const float h = P.h;
    const F2 half = bc2(0.5f * h), full = bc2(h), sixth = bc2(h / 6.f);
    P3 c{bc2(0.f), bc2(0.f), bc2(0.f)};    // Kahan compensation of the position sums
    float sfree[2] = {0.f, 0.f};           // sphere / half-space free distance budgets
    float mfree[2] = {0.f, 0.f};           // mesh free distance budgets (MESH)
    float bfree[2] = {0.f, 0.f};           // bounds-box distance budgets (RR_BOUNDS_BUDGET)
    for (;;) {
        if (!__any_sync(kFull, act[0] || act[1])) break;
        cnt.lane_slots += 2;
        int nj[2] = {0, 0};
        uint32_t um = 0u;
        if constexpr (KIND == kBumps) {
            uint32_t lmo = 0u;
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                uint32_t lm = 0u;
                unsigned cell = 0;
                if (act[r]) {
                    if (P.cull) {
                        cell = cell_of(P, ray_of(p, r));
                        lm = __ldg(P.cull_masks + cell);
                    } else {
                        lm = P.all_mask;
                    }
                    if (P.skip && lm == 0u) {
                        const int k = __ldg(P.skip_k + cell);
                        if (k >= 2) nj[r] = jump_steps<PASS>(P, ray_of(p, r), ray_of(v, r), k, step[r], qq[r], light_d[r], kShadow);
                    }
                }
                lmo |= nj[r] ? 0u : lm;
#if RR_COUNT_OWN_MASK
                if (act[r] && !nj[r]) cnt.bump_evals += 4u * __popc(lm);   // diagnostics: per-ray N_eff
#endif
            }
            um = __reduce_or_sync(kFull, lmo);
#if !RR_COUNT_OWN_MASK
#pragma unroll
            for (int r = 0; r < 2; ++r)
                if (act[r] && !nj[r]) cnt.bump_evals += 4u * __popc(um);
#endif
        }
        P3 dp, vn;
        float vld[2] = {3.0e38f, 3.0e38f};                  // diffeo chains: min |det J| of the step
        const bool jw0 = nj[0] != 0 || !act[0], jw1 = nj[1] != 0 || !act[1];
        if (KIND == kBumps && __all_sync(kFull, jw0 && jw1)) {   // whole warp jumps: no integration
            dp = P3{bc2(0.f), bc2(0.f), bc2(0.f)};
            vn = v;
        } else if constexpr (KIND == kDiffeo) {
            twist_rk4_x2(p, v, half, full, sixth, dp, vn);
        } else if constexpr (KIND == kDiffeoChain) {        // RK4 over the packed jet fold
            P3 sx{bc2(0.f), bc2(0.f), bc2(0.f)}, sv{bc2(0.f), bc2(0.f), bc2(0.f)};
            P3 ps = p, vs = v;
#pragma unroll 1
            for (int st = 0; st < 4; ++st) {   // rolled: one copy of the fold (instruction cache)
                const P3 a = accel_diffeo_x2<NB>(P, ps, vs, vld);
                const F2 wgt = bc2((st == 0 || st == 3) ? 1.f : 2.f);
                sx = P3{fma2(wgt, vs.x, sx.x), fma2(wgt, vs.y, sx.y), fma2(wgt, vs.z, sx.z)};
                sv = P3{fma2(wgt, a.x, sv.x), fma2(wgt, a.y, sv.y), fma2(wgt, a.z, sv.z)};
                const F2 cc = st < 2 ? half : full;
                ps = P3{fma2(cc, vs.x, p.x), fma2(cc, vs.y, p.y), fma2(cc, vs.z, p.z)};
                vs = P3{fma2(cc, a.x, v.x), fma2(cc, a.y, v.y), fma2(cc, a.z, v.z)};
            }
            dp = P3{mul2(sixth, sx.x), mul2(sixth, sx.y), mul2(sixth, sx.z)};
            vn = P3{fma2(sixth, sv.x, v.x), fma2(sixth, sv.y, v.y), fma2(sixth, sv.z, v.z)};
        } else {                                             // RK4 (integrate.hpp:63-93)
            P3 sx{bc2(0.f), bc2(0.f), bc2(0.f)}, sv{bc2(0.f), bc2(0.f), bc2(0.f)};
            P3 ps = p, vs = v;
            auto stage = [&](int st) {
                const P3 a = accel_bumps_x2<NB, PASS != kPassShade && RR_X2_SCALAR_CONSTS_LIT>(P, um, ps, vs);
                const F2 wgt = bc2((st == 0 || st == 3) ? 1.f : 2.f);
                sx = P3{fma2(wgt, vs.x, sx.x), fma2(wgt, vs.y, sx.y), fma2(wgt, vs.z, sx.z)};
                sv = P3{fma2(wgt, a.x, sv.x), fma2(wgt, a.y, sv.y), fma2(wgt, a.z, sv.z)};
                const F2 cc = st < 2 ? half : full;
                ps = P3{fma2(cc, vs.x, p.x), fma2(cc, vs.y, p.y), fma2(cc, vs.z, p.z)};
                vs = P3{fma2(cc, a.x, v.x), fma2(cc, a.y, v.y), fma2(cc, a.z, v.z)};
            };
            // unlit frames: the four stages unrolled (four bump loops); the lit
            // launch carries two march copies, RR_X2_RK4_UNROLL_LIT picks its form
            constexpr bool kUnrollStages = PASS == kPassShade ? RR_X2_RK4_UNROLL
                                         : PASS == kPassShadow ? RR_X2_RK4_UNROLL_SHADOW
                                                               : RR_X2_RK4_UNROLL_LIT;
            if constexpr (kUnrollStages) {
#pragma unroll
                for (int st = 0; st < 4; ++st) stage(st);
            } else {
#pragma unroll 1
                for (int st = 0; st < 4; ++st) stage(st);   // one call site: the bump block is inlined once
            }
            dp = P3{mul2(sixth, sx.x), mul2(sixth, sx.y), mul2(sixth, sx.z)};
            vn = P3{fma2(sixth, sv.x, v.x), fma2(sixth, sv.y, v.y), fma2(sixth, sv.z, v.z)};
        }
        if (KIND == kBumps && (nj[0] | nj[1])) {            // straight jumps of nj steps
            const F2 hn = mk2(h * (float)nj[0], h * (float)nj[1]);
            const P3 dj{mul2(hn, v.x), mul2(hn, v.y), mul2(hn, v.z)};
            const bool j0 = nj[0] != 0, j1 = nj[1] != 0;
            dp = P3{sel2(j0, j1, dj.x, dp.x), sel2(j0, j1, dj.y, dp.y), sel2(j0, j1, dj.z, dp.z)};
            vn = P3{sel2(j0, j1, v.x, vn.x), sel2(j0, j1, v.y, vn.y), sel2(j0, j1, v.z, vn.z)};
        }
        // compensated position update: pn = p + dp carrying the rounding error
#if RR_X2_KAHAN
        const P3 yv{sub2(dp.x, c.x), sub2(dp.y, c.y), sub2(dp.z, c.z)};
        const P3 pn{add2(p.x, yv.x), add2(p.y, yv.y), add2(p.z, yv.z)};
        c = P3{sub2(sub2(pn.x, p.x), yv.x), sub2(sub2(pn.y, p.y), yv.y), sub2(sub2(pn.z, p.z), yv.z)};
#else
        (void)c;
        const P3 pn{add2(p.x, dp.x), add2(p.y, dp.y), add2(p.z, dp.z)};
#endif
        // chord tests (scene.cpp:99-109): analytic primitives per ray; with
        // meshes, the rays whose chord leaves their free ball are collected
        // and the warp runs the BVH tests over that compacted list (one
        // traversal per iteration for every thread with work, whichever of
        // its two rays needs it) instead of once per ray slot
        bool hit[2] = {false, false};
        float sh[2] = {0.f, 0.f};
        float clen[2] = {0.f, 0.f};                     // conservative chord lengths
        int primr[2] = {-1, -1}, hidr[2] = {0, 0}, mrec[2] = {0, 0};
        if constexpr (MESH) {
            unsigned pend = 0u;
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                if (!act[r]) continue;
                const F3 a = ray_of(p, r), b = ray_of(pn, r);
                float md = 0.f;
                int mr = 0;
                hit[r] = intersect<false>(P, a, b, sh[r], primr[r], hidr[r], md, mr, sfree[r], clen[r]);
                const float len = clen[r];
                float gd;
                if (len < mfree[r]) mfree[r] -= len;     // the chord stays inside the free ball
                else if ((gd = mesh_grid_free(P, a)) > len) mfree[r] = gd - len;   // distance grid
                else pend |= 1u << r;
            }
            while (__any_sync(kFull, pend != 0u)) {
                if (pend) {
                    const int r = (pend & 1u) ? 0 : 1;
                    pend &= pend - 1u;
                    const F3 a = r ? ray_of(p, 1) : ray_of(p, 0);
                    const F3 b = r ? ray_of(pn, 1) : ray_of(pn, 0);
                    const F3 d = f3(b.x - a.x, b.y - a.y, b.z - a.z);
                    bool hv = r ? hit[1] : hit[0];
                    float sb = r ? sh[1] : sh[0];
                    int pr = r ? primr[1] : primr[0], hd = r ? hidr[1] : hidr[0];
                    int mc = 0;
                    float mf = 0.f;
                    mesh_part(P, a, d, 0.f, hv, sb, pr, hd, mc, mf);
                    if (r) { hit[1] = hv; sh[1] = sb; primr[1] = pr; hidr[1] = hd; mrec[1] = mc; mfree[1] = mf; }
                    else { hit[0] = hv; sh[0] = sb; primr[0] = pr; hidr[0] = hd; mrec[0] = mc; mfree[0] = mf; }
                }
            }
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            if (!act[r]) continue;
            const F3 a = ray_of(p, r), b = ray_of(pn, r);
            const int nsub = nj[r] ? nj[r] : 1;
            cnt.steps_integrated += 1;
            cnt.jumps += nj[r] ? 1u : 0u;
            if constexpr (KIND == kDiffeoChain) {
                if (!(vld[r] > 1e-14f)) {                   // kernel_impl.hpp:54-61: Failed
                    act[r] = false;
                    if (kShadow) {
                        status[r] = 0;
                        steps[r] = step[r];
                    } else {
                        if (kHits && !RR_X2_HITS_STAGED) {
                            RayResult res{2, -1, step[r], 0.f, f3(0.f, 0.f, 0.f), f3(0.f, 0.f, 0.f)};
                            emit_primary<kPassHits>(P, L, unit, r, res);
                        } else {
                            stg->tp[r * kUnit + lane] = make_float4(0.f, 0.f, 0.f, 0.f);
                            stg->sp[r * kUnit + lane] = make_int2(2, step[r]);
                        }
                        us.ref_steps += (unsigned)step[r];
                    }
                    continue;
                }
            }
            float s = sh[r];
            int prim = primr[r], hid = hidr[r];
            if constexpr (!MESH) {   // analytic primitives only: test and consume in one pass
                float md = 0.f;
                int mr = 0;
                hit[r] = intersect<false>(P, a, b, s, prim, hid, md, mr, sfree[r], clen[r]);
            }
            if (hit[r]) {                                    // kernel_impl.hpp:63-76
                const F3 pt = f3(fmaf(s, b.x - a.x, a.x), fmaf(s, b.y - a.y, a.y), fmaf(s, b.z - a.z, a.z));
                const float sj = s * (float)nsub;            // hit position in reference steps
                const int sub = min((int)sj, nsub - 1);
                if (kShadow) {
                    const F3 rr = f3(pt.x - qq[r].x, pt.y - qq[r].y, pt.z - qq[r].z);
                    status[r] = (rr.x * rr.x + rr.y * rr.y + rr.z * rr.z) < dd[r] ? 0 : 1;
                    steps[r] = step[r] + sub + 1;
                } else {
                    const float th = ((float)step[r] + sj) * h;
                    const int nst = step[r] + sub + 1;
                    if (kHits && !RR_X2_HITS_STAGED) {
                        RayResult res{1, prim, nst, th, pt, f3(0.f, 0.f, 0.f)};
                        res.normal = hit_normal(P, hid, s, a, b, pt, mrec[r]);
                        emit_primary<kPassHits>(P, L, unit, r, res);
                    } else {
                        if (kHits) {
                            stg->chord[r * kUnit + lane] = make_float4(a.x, a.y, a.z, s);
                            stg->chord[(2 + r) * kUnit + lane] =
                                make_float4(b.x, b.y, b.z, __int_as_float(hid | (mrec[r] << 12)));
                        }
                        stg->tp[r * kUnit + lane] = make_float4(th, pt.x, pt.y, pt.z);
                        stg->sp[r * kUnit + lane] = make_int2(1 | ((prim + 1) << 8), nst);
                    }
                    us.ref_steps += (unsigned)nst;
                }
                act[r] = false;
            } else if (kShadow &&
                       (b.x - qq[r].x) * (b.x - qq[r].x) + (b.y - qq[r].y) * (b.y - qq[r].y) +
                               (b.z - qq[r].z) * (b.z - qq[r].z) >= dd[r]) {
                status[r] = 1;                               // reached the light's sphere
                steps[r] = step[r] + nsub;
                act[r] = false;
            } else {
                step[r] += nsub;
                bool out;                                    // kernel_impl.hpp:77-82
                if constexpr (RR_BOUNDS_BUDGET && KIND == kDiffeo) {
                    // exact test only once the chords since the last one have
                    // used up the point's distance to the bounds box (same
                    // outcome; measured a win only on the single twist, whose
                    // step is cheap: C4 6.56 -> 6.47 ms, r2z_bounds_budget_ab.log)
                    bfree[r] -= clen[r];
                    if (bfree[r] > 0.f) {
                        out = false;
                    } else {
                        out = !inside_bounds(P, b);
                        bfree[r] = out ? 0.f : bounds_free(P, b);
                    }
                } else {
                    out = !inside_bounds(P, b);
                }
                if (out || step[r] >= P.max_steps) {         // kernel_impl.hpp:87-91
                    const int nst = out ? step[r] : P.max_steps;
                    act[r] = false;
                    if (kShadow) {
                        status[r] = 1;
                        steps[r] = nst;
                    } else {
                        if (kHits && !RR_X2_HITS_STAGED) {
                            RayResult res{0, -1, nst, 0.f, f3(0.f, 0.f, 0.f), f3(0.f, 0.f, 0.f)};
                            emit_primary<kPassHits>(P, L, unit, r, res);
                        } else {
                            stg->tp[r * kUnit + lane] = make_float4(0.f, 0.f, 0.f, 0.f);
                            stg->sp[r * kUnit + lane] = make_int2(0, nst);
                        }
                        us.ref_steps += (unsigned)nst;
                    }
                }
                continue;
            }
            step[r] += nsub;
        }
        p = pn;
        v = vn;
    }
}

// RGB8 of a one-ray unit's 8x4 micro-tile: when every lane writes its pixel
// and the rows are 8-B aligned (L.vec8), the 4 x 24-byte block is assembled
// in shared memory and stored as 12 8-byte words (sector-friendly over
// PCIe/NVLink for UVA / peer frames), else byte-wise.
__device__ __forceinline__ void store_unit_rgb(const DevLaunch& L, int lane, unsigned long long pix,
                                               uint32_t rgb, bool writer, uint32_t* smem24) {
    if (L.vec8 && __all_sync(kFull, writer)) {
        uint8_t* sb = reinterpret_cast<uint8_t*>(smem24);
        const int off = (lane >> 3) * 24 + (lane & 7) * 3;
        sb[off] = (uint8_t)(rgb & 0xff);
        sb[off + 1] = (uint8_t)((rgb >> 8) & 0xff);
        sb[off + 2] = (uint8_t)((rgb >> 16) & 0xff);
        __syncwarp();
        const unsigned long long rowpix = __shfl_sync(kFull, pix, (lane / 3 & 3) * 8);
        if (lane < 12) {
            RR_CHECK(rowpix + kMicroW <= L.out_pixels && ((3 * rowpix) & 7) == 0, "rgb micro-tile row");
            *reinterpret_cast<uint2*>(L.rgb + 3 * rowpix + 8 * (lane % 3)) =
                reinterpret_cast<const uint2*>(smem24)[lane];
        }
        __syncwarp();
        return;
    }
    if (writer) {
        RR_CHECK(pix < L.out_pixels, "rgb pixel index (one-ray)");
        uint8_t* dst = L.rgb + 3 * pix;
        dst[0] = (uint8_t)(rgb & 0xff);
        dst[1] = (uint8_t)((rgb >> 8) & 0xff);
        dst[2] = (uint8_t)((rgb >> 16) & 0xff);
    }
}

template <int KIND, int NB, int SCHEME, int PASS, bool MESH>
__global__ void __launch_bounds__(kThreads, SCHEME == 2 ? RR_MIN_BLOCKS_RK23
                                         : (MESH ? RR_MIN_BLOCKS_MESH : RR_MIN_BLOCKS))
march_kernel(const __grid_constant__ DevParams P, const __grid_constant__ DevLaunch L) {
    const int lane = threadIdx.x & 31;
    __shared__ uint32_t s_rgb[kThreads / 32][24];   // 8x4 RGB8 micro-tile per warp
    __shared__ unsigned long long s_acc[kThreads / 32][8];   // the warp's stat sums (lane 0)
    unsigned long long* acc = s_acc[threadIdx.x >> 5];
    if (lane == 0)
        for (int k = 0; k < 8; ++k) acc[k] = 0ull;
    // Euclidean units are cheap (straight jumps): the unit fetch's returning
    // atomic is issued one unit ahead, so its latency overlaps the current unit
    constexpr bool kPrefetch = KIND == kEuclid && RR_EUCLID_PREFETCH;
    unsigned next = 0;
    if (kPrefetch && lane == 0) next = atomicAdd(L.counter, 1u);
    for (;;) {
        unsigned unit = 0;
        if constexpr (kPrefetch) {
            unit = __shfl_sync(kFull, next, 0);
            if (unit >= L.n_units) break;
            if (lane == 0) next = atomicAdd(L.counter, 1u);
        } else {
            if (lane == 0) unit = atomicAdd(L.counter, 1u);
            unit = __shfl_sync(kFull, unit, 0);
            if (unit >= L.n_units) break;
        }

        bool live;
        F3 pos, dir;
        int px = 0, py = 0, lx = 0, ly = 0;
        unsigned long long ray_index = 0, tile_k = 0, pix = 0;
        if (L.mode == kModeRays) {
            ray_index = (unsigned long long)unit * kUnit + lane;
            live = ray_index < L.n_rays;
            if (live) {
                const double* r = L.rays + 6 * ray_index;
                pos = f3((float)r[0], (float)r[1], (float)r[2]);
                dir = f3((float)r[3], (float)r[4], (float)r[5]);
            } else {
                pos = dir = f3(0.f, 0.f, 0.f);
            }
        } else {
            // shadow pass: a unit is 32/lpp pixels of a micro-tile x lpp lights
            const unsigned mt = PASS == kPassShadow ? unit / L.lpp : unit;
            const int sub = PASS == kPassShadow ? (int)(unit % L.lpp) : 0;
            const int ppu = PASS == kPassShadow ? kUnit / L.lpp : kUnit;
            const int idx = sub * ppu + lane % ppu;          // pixel within the micro-tile
            tile_k = mt / L.micro_per_tile;
            const unsigned micro = mt % L.micro_per_tile;
            const unsigned tile = L.shard + (unsigned)tile_k * L.n_shards;
            const int tx = tile % L.tiles_x, ty = tile / L.tiles_x;
            const int mpr = L.tile_w / kMicroW;
            lx = (micro % mpr) * kMicroW + (idx & 7);
            ly = (micro / mpr) * kMicroH + (idx >> 3);
            px = tx * L.tile_w + lx;
            py = ty * L.tile_h + ly;
            live = px < L.width && py < L.height;
            // output index: row-major frame, or tile-major shard buffer
            pix = L.mode == kModeFrame ? (unsigned long long)py * L.width + px
                                       : tile_k * L.tile_w * L.tile_h + (unsigned long long)ly * L.tile_w + lx;
            if (PASS != kPassShadow) {
                if (live) raygen(L.cam, px, py, L.width, L.height, pos, dir);
                else pos = dir = f3(0.f, 0.f, 0.f);
            }
        }

        LaneCounters cnt{0u, 0u, 0u, 0u};
        unsigned ref_steps = 0, errs = 0, shadow_steps = 0;
        bool pad_writer = true;
        if constexpr (PASS == kPassShadow) {
            // ---- EXTENSION: shadow geodesics.  Lane = (pixel, light): lpp lights
            // of 32/lpp pixels march together; contributions are summed across
            // the lanes of a pixel; light groups beyond lpp loop.
            const int ppu = kUnit / L.lpp;
            const int li = lane / ppu;
            HitRec hr{};
            RR_CHECK(!live || pix < L.out_pixels, "hit record read (one-ray)");
            if (live) hr = L.hits[pix];
            const bool hit = live && (hr.status == 1);
            const F3 q = f3(hr.p[0], hr.p[1], hr.p[2]);
            const F3 n = f3(hr.n[0], hr.n[1], hr.n[2]);
            float contrib = 0.f;
            for (int lg = 0; lg < P.n_lights; lg += L.lpp) {
                const int l = lg + li;
                const DevLight& Lt = P.lights[l < P.n_lights ? l : 0];
                const F3 D = f3(Lt.pos[0] - q.x, Lt.pos[1] - q.y, Lt.pos[2] - q.z);
                const float dist2 = D.x * D.x + D.y * D.y + D.z * D.z;
                const float lam = (n.x * D.x + n.y * D.y + n.z * D.z) * rsqrtf(dist2);
                bool want = hit && l < P.n_lights && lam > 0.f;
                F3 x0 = f3(0.f, 0.f, 0.f), v0 = f3(0.f, 0.f, 0.f);
                if (want) {
                    x0 = f3(fmaf(kShadowEps, n.x, q.x), fmaf(kShadowEps, n.y, q.y),
                            fmaf(kShadowEps, n.z, q.z));
                    float g[6];
                    bool ok;
                    metric_at(P, x0, g, ok);
                    const float n2 = g[0] * D.x * D.x + g[3] * D.y * D.y + g[5] * D.z * D.z +
                                     2.f * (g[1] * D.x * D.y + g[2] * D.x * D.z + g[4] * D.y * D.z);
                    const float inv = rsqrtf(n2);
                    v0 = f3(D.x * inv, D.y * inv, D.z * inv);
                    want = ok;
                }
                const RayResult sr = march_unit<KIND, NB, SCHEME, kPassShadow, MESH>(P, want, x0, v0, cnt, q, dist2);
                if (want) shadow_steps += (unsigned)sr.steps;   // reference-equivalent steps
                if (want && sr.status == 1) contrib = fmaf(Lt.intensity, lam, contrib);
            }
            // sum over the lanes of a pixel (same lane % ppu), in light order
            for (int o = ppu; o < kUnit; o <<= 1) contrib += __shfl_xor_sync(kFull, contrib, o);
            uint32_t rgbw = 0u;
            if (live && li == 0) rgbw = shade_rgb(P, hr.status, hr.t, q, P.ambient + contrib);
            pad_writer = li == 0;     // one writer per pixel for the tile padding
            if (L.lpp == 1) {
                store_unit_rgb(L, lane, pix, rgbw, live || L.mode == kModeTiles, s_rgb[threadIdx.x >> 5]);
                pad_writer = false;   // the padding went with the block
            } else if (live && li == 0) {
                uint8_t* dst = L.rgb + 3 * pix;
                dst[0] = (uint8_t)(rgbw & 0xff);
                dst[1] = (uint8_t)((rgbw >> 8) & 0xff);
                dst[2] = (uint8_t)((rgbw >> 16) & 0xff);
            }
        } else {
            const RayResult r = march_unit<KIND, NB, SCHEME, PASS, MESH>(P, live, pos, dir, cnt);
            ref_steps = live ? (unsigned)r.steps : 0u;
            errs = (live && r.status == 2) ? 1u : 0u;
            if (live) {
                // render::PixelOutcome: batch mode always; frames when the
                // launch carries an outcome sink (row-major pixel index)
                if (L.outcomes)
                    write_outcome(L.outcomes,
                                  L.mode == kModeRays ? ray_index
                                                      : (unsigned long long)py * L.width + px,
                                  r.status, r.prim, r.point, r.t, r.steps, L.n_outcomes);
                if (L.mode == kModeRays) {
                } else if constexpr (PASS == kPassHits) {
                    RR_CHECK(pix < L.out_pixels, "hit record index (one-ray)");
                    HitRec hr;
                    hr.p[0] = r.point.x;
                    hr.p[1] = r.point.y;
                    hr.p[2] = r.point.z;
                    hr.t = r.t;
                    hr.n[0] = r.normal.x;
                    hr.n[1] = r.normal.y;
                    hr.n[2] = r.normal.z;
                    hr.status = r.status;
                    L.hits[pix] = hr;
                }
            }
            if (L.mode != kModeRays && PASS == kPassShade) {
                // the micro-tile's pixels (zero partial-tile padding in tile mode)
                const uint32_t rgbw = live ? shade_rgb(P, r.status, r.t, r.point) : 0u;
                store_unit_rgb(L, lane, pix, rgbw, live || L.mode == kModeTiles, s_rgb[threadIdx.x >> 5]);
            }
        }
        if (PASS == kPassShadow && !live && pad_writer && L.mode == kModeTiles) {
            uint8_t* dst = L.rgb + 3 * pix;
            dst[0] = dst[1] = dst[2] = 0;
        }
        // per-unit counters: one REDUX per counter, summed per warp in shared
        // memory and flushed with one 64-bit atomic per counter when the warp
        // leaves the loop (per-unit atomics on the 11 shared stat words
        // serialised in L2 for launches of cheap units)
        const unsigned steps = __reduce_add_sync(kFull, ref_steps);
        const unsigned nerr = __reduce_add_sync(kFull, errs);
        const unsigned integ = __reduce_add_sync(kFull, cnt.steps_integrated);
        const unsigned evals = __reduce_add_sync(kFull, cnt.bump_evals);
        const unsigned nr = __reduce_add_sync(kFull, (live && PASS != kPassShadow) ? 1u : 0u);
        const unsigned shs = __reduce_add_sync(kFull, shadow_steps);
        const unsigned slots = __reduce_add_sync(kFull, cnt.lane_slots);
        const unsigned jmp = __reduce_add_sync(kFull, cnt.jumps);
        if (lane == 0) {
            acc[0] += steps;
            acc[1] += nerr;
            acc[2] += integ;
            acc[3] += evals;
            acc[4] += nr;
            acc[5] += shs;
            acc[6] += slots;
            acc[7] += jmp;
        }
    }
    if (lane == 0) {
        if (acc[7]) atomicAdd(L.stats + (PASS == kPassShadow ? 9 : 8), acc[7]);
        if (acc[2] && PASS == kPassShadow) atomicAdd(L.stats + 10, acc[2]);
        if (acc[0]) atomicAdd(L.stats + 0, acc[0]);
        if (acc[1]) atomicAdd(L.stats + 1, acc[1]);
        if (acc[2]) atomicAdd(L.stats + 2, acc[2]);
        if (acc[3]) atomicAdd(L.stats + 3, acc[3]);
        if (acc[4]) atomicAdd(L.stats + 4, acc[4]);
        if (acc[5]) atomicAdd(L.stats + 5, acc[5]);
        if (acc[6]) atomicAdd(L.stats + (PASS == kPassShadow ? 7 : 6), acc[6]);
    }
    // Sharded frame mode may write into another GPU's frame (peer/IPC mapping):
    // make the stores visible system-wide before the kernel retires, ahead of
    // the cross-rank synchronisation that hands the frame to its owner.
    if (L.mode == kModeFrame && L.n_shards > 1) __threadfence_system();
}


// ---------------------------------------------------------------------------
// Ray-pair frame kernel (Gaussian bumps, RK4, no meshes; frame and tile
// modes).  A unit is two consecutive micro-tiles of march_kernel's order
// (ray 0 of a thread in micro-tile 2u, ray 1 in 2u+1, same lane position),
// so tiles remain unions of units (byte-identical frames across shard
// counts).  L.n_units counts micro-tiles; the kernel serves (n+1)/2 units.
// With lights the shadow pass marches light by light (lpp = 1).
__device__ __forceinline__ void pixel_of(const DevLaunch& L, unsigned mt, int lane, bool& inrange,
                                         bool& live, int& px, int& py, unsigned long long& pix) {
    inrange = mt < L.n_units;
    const unsigned m = inrange ? mt : 0u;
    const unsigned long long tile_k = m / L.micro_per_tile;
    const unsigned micro = m % L.micro_per_tile;
    const unsigned tile = L.shard + (unsigned)tile_k * L.n_shards;
    const int tx = tile % L.tiles_x, ty = tile / L.tiles_x;
    const int mpr = L.tile_w / kMicroW;
    const int lx = (micro % mpr) * kMicroW + (lane & 7);
    const int ly = (micro / mpr) * kMicroH + (lane >> 3);
    px = tx * L.tile_w + lx;
    py = ty * L.tile_h + ly;
    live = inrange && px < L.width && py < L.height;
    pix = L.mode == kModeFrame ? (unsigned long long)py * L.width + px
                               : tile_k * L.tile_w * L.tile_h + (unsigned long long)ly * L.tile_w + lx;
}

// Output of a terminated primary ray of a kPassHits pair unit (pixel
// recomputed from the unit, so no output addresses stay live through the
// march): the 32-B hit record for the shadow work, plus the PixelOutcome
// record when the launch carries an outcome sink.
template <int PASS>
__device__ __forceinline__ void emit_primary(const DevParams& P, const DevLaunch& L, unsigned unit,
                                             int r, const RayResult& res) {
    bool inr, live;
    int px, py;
    unsigned long long pix;
    pixel_of(L, 2 * unit + r, threadIdx.x & 31, inr, live, px, py, pix);
    if constexpr (PASS == kPassHits) {
        HitRec h;
        h.p[0] = res.point.x;
        h.p[1] = res.point.y;
        h.p[2] = res.point.z;
        h.t = res.t;
        h.n[0] = res.normal.x;
        h.n[1] = res.normal.y;
        h.n[2] = res.normal.z;
        h.status = res.status;
        RR_CHECK(live && pix < L.out_pixels, "hit record index");
        L.hits[pix] = h;
        if (L.outcomes)
            write_outcome(L.outcomes, (unsigned long long)py * L.width + px, res.status, res.prim,
                          res.point, res.t, res.steps, L.n_outcomes);
    }
}

// Per-warp accounting of one work unit, flushed with one atomic per field.
__device__ __forceinline__ void flush_unit_stats(const DevLaunch& L, const UnitStats& us, int lane,
                                                 bool shadow) {
    const unsigned steps = __reduce_add_sync(kFull, us.ref_steps);
    const unsigned nerr = __reduce_add_sync(kFull, us.errs);
    const unsigned integ = __reduce_add_sync(kFull, us.cnt.steps_integrated);
    const unsigned evals = __reduce_add_sync(kFull, us.cnt.bump_evals);
    const unsigned nr = __reduce_add_sync(kFull, us.nrays);
    const unsigned shs = __reduce_add_sync(kFull, us.shadow_steps);
    const unsigned slots = __reduce_add_sync(kFull, us.cnt.lane_slots);
    const unsigned jmp = __reduce_add_sync(kFull, us.cnt.jumps);
    if (lane == 0) {
        if (jmp) atomicAdd(L.stats + (shadow ? 9 : 8), (unsigned long long)jmp);
        if (integ && shadow) atomicAdd(L.stats + 10, (unsigned long long)integ);
        if (steps) atomicAdd(L.stats + 0, (unsigned long long)steps);
        if (nerr) atomicAdd(L.stats + 1, (unsigned long long)nerr);
        if (integ) atomicAdd(L.stats + 2, (unsigned long long)integ);
        if (evals) atomicAdd(L.stats + 3, (unsigned long long)evals);
        if (nr) atomicAdd(L.stats + 4, (unsigned long long)nr);
        if (shs) atomicAdd(L.stats + 5, (unsigned long long)shs);
        if (slots) atomicAdd(L.stats + (shadow ? 7 : 6), (unsigned long long)slots);
    }
}

// RGB8 of the 64 pixels of a ray-pair unit (rgb[r] = lane's pixel of
// micro-tile 2 unit + r, packed r | g << 8 | b << 16).  When the launch
// allows it (L.vec16: 16-B aligned rows, micro-tiles 2u and 2u+1 side by
// side) and the 16x4 block lies inside the frame, the block is assembled in
// shared memory and written as 12 16-byte stores (4 rows x 48 bytes) — one
// sector-sized transaction per 16 bytes instead of 192 byte stores, which
// matters most when the frame is pinned host memory (UVA) or a peer GPU's
// frame (NVLink).  Otherwise pixels are stored byte-wise; in tile mode the
// padding pixels of partial tiles are zeroed either way.
__device__ __forceinline__ void store_pair_rgb(const DevLaunch& L, unsigned unit, int lane,
                                               const uint32_t (&rgb)[2], PairStage* stg) {
    bool inr[2], live[2];
    int px[2], py[2];
    unsigned long long pix[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) pixel_of(L, 2 * unit + r, lane, inr[r], live[r], px[r], py[r], pix[r]);
    const int px0 = __shfl_sync(kFull, px[0], 0), py0 = __shfl_sync(kFull, py[0], 0);
    const bool full = L.vec16 && inr[1] &&
                      (L.mode == kModeTiles || (px0 + 2 * kMicroW <= L.width && py0 + kMicroH <= L.height));
    if (full) {
        uint8_t* sb = reinterpret_cast<uint8_t*>(stg->rgb);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int off = (lane >> 3) * 48 + (r * kMicroW + (lane & 7)) * 3;
            sb[off] = (uint8_t)(rgb[r] & 0xff);
            sb[off + 1] = (uint8_t)((rgb[r] >> 8) & 0xff);
            sb[off + 2] = (uint8_t)((rgb[r] >> 16) & 0xff);
        }
        __syncwarp();
        const unsigned long long rowpix = __shfl_sync(kFull, pix[0], (lane / 3 & 3) * 8);
        if (lane < 12) {
            RR_CHECK(rowpix + 2 * kMicroW <= L.out_pixels && ((3 * rowpix) & 15) == 0, "rgb block row");
            const uint4 v = reinterpret_cast<const uint4*>(stg->rgb)[lane];
            *reinterpret_cast<uint4*>(L.rgb + 3 * rowpix + 16 * (lane % 3)) = v;
        }
        __syncwarp();
        return;
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        if (live[r] || (inr[r] && L.mode == kModeTiles)) {
            RR_CHECK(pix[r] < L.out_pixels, "rgb pixel index");
            uint8_t* dst = L.rgb + 3 * pix[r];
            const uint32_t c = live[r] ? rgb[r] : 0u;
            dst[0] = (uint8_t)(c & 0xff);
            dst[1] = (uint8_t)((c >> 8) & 0xff);
            dst[2] = (uint8_t)((c >> 16) & 0xff);
        }
    }
}

// Primary rays of ray-pair unit `unit` (64 pixels: micro-tiles 2 unit, 2 unit
// + 1; or, in batch mode, rays 64 unit .. 64 unit + 63): raygen (or the
// caller's RayStart records), march, and either the fused shading
// (kPassShade: from the warp's PairStage, plus the PixelOutcome records when
// the launch carries an outcome sink) or hit records for the shadow work
// (kPassHits).
template <int KIND, int NB, int PASS, bool MESH>
__device__ __forceinline__ void pair_primary(const DevParams& P, const DevLaunch& L, unsigned unit,
                                             int lane, UnitStats& us, PairStage* stg) {
    bool live[2];
    F3 pos[2], dir[2];
    const bool rays = L.mode == kModeRays;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        pos[r] = dir[r] = f3(0.f, 0.f, 0.f);
        if (rays) {
            const unsigned long long idx = (2ull * unit + r) * kUnit + lane;
            live[r] = idx < L.n_rays;
            if (live[r]) {
                const double* q = L.rays + 6 * idx;
                pos[r] = f3((float)q[0], (float)q[1], (float)q[2]);
                dir[r] = f3((float)q[3], (float)q[4], (float)q[5]);
            }
        } else {
            bool inr;
            int px, py;
            unsigned long long pix;
            pixel_of(L, 2 * unit + r, lane, inr, live[r], px, py, pix);
            if (live[r]) raygen(L.cam, px, py, L.width, L.height, pos[r], dir[r]);
        }
        us.nrays += live[r] ? 1u : 0u;
    }
    int st[2], stp[2];
    march_pair<KIND, NB, PASS, MESH>(P, live[0], live[1], pair_of(pos[0], pos[1]), pair_of(dir[0], dir[1]),
                         us, L, unit, st, stp, stg);
    if constexpr (PASS == kPassHits && RR_X2_HITS_STAGED) {
        // hit records (normal, 32-B HitRec) + outcome records from the stage
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            if (!live[r] || rays) continue;
            const float4 tp = stg->tp[r * kUnit + lane];
            const int2 sp = stg->sp[r * kUnit + lane];
            const int status = sp.x & 0xff;
            RayResult res{status, (sp.x >> 8) - 1, sp.y, tp.x, f3(tp.y, tp.z, tp.w), f3(0.f, 0.f, 0.f)};
            if (status == 1) {
                const float4 ca = stg->chord[r * kUnit + lane];
                const float4 cb = stg->chord[(2 + r) * kUnit + lane];
                const int hm = __float_as_int(cb.w);
                res.normal = hit_normal(P, hm & 0xfff, ca.w, f3(ca.x, ca.y, ca.z), f3(cb.x, cb.y, cb.z),
                                        res.point, hm >> 12);
            } else {
                res.prim = -1;
            }
            emit_primary<kPassHits>(P, L, unit, r, res);
        }
        __syncwarp();
    }
    if constexpr (PASS == kPassShade) {
        __syncwarp();
        uint32_t rgb[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            rgb[r] = 0u;
            if (!live[r]) continue;
            const float4 tp = stg->tp[r * kUnit + lane];
            const int2 sp = stg->sp[r * kUnit + lane];
            const int status = sp.x & 0xff;
            const F3 pt = f3(tp.y, tp.z, tp.w);
            us.errs += status == 2 ? 1u : 0u;
            rgb[r] = shade_rgb(P, status, tp.x, pt);
            if (L.outcomes) {
                unsigned long long idx;
                if (rays) {
                    idx = (2ull * unit + r) * kUnit + lane;
                } else {
                    bool inr, lv;
                    int px, py;
                    unsigned long long pix;
                    pixel_of(L, 2 * unit + r, lane, inr, lv, px, py, pix);
                    idx = (unsigned long long)py * L.width + px;
                }
                write_outcome(L.outcomes, idx, status, (sp.x >> 8) - 1, pt, tp.x, sp.y, L.n_outcomes);
            }
        }
        if (!rays) store_pair_rgb(L, unit, lane, rgb, stg);
        __syncwarp();
    }
}

// ---- EXTENSION: shadow geodesics (oracle/rro.c shadow_march) of ray-pair
// unit `unit` toward light `l`.  Each (unit, light) is its own work item, so
// the expensive shadow work is split finely across warps; the visibility
// byte of every (pixel, light) is published and the unit's LAST light to
// finish (per-unit counter L.done) shades its 64 pixels, summing the lit
// contributions in light order (shade_lit in oracle/rro.c).
template <int KIND, int NB, bool MESH>
__device__ __forceinline__ void pair_shadow(const DevParams& P, const DevLaunch& L, unsigned unit,
                                            int l, int nl, int lane, UnitStats& us, PairStage* stg) {
    bool inr[2], live[2];
    int px[2], py[2];
    unsigned long long pix[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) pixel_of(L, 2 * unit + r, lane, inr[r], live[r], px[r], py[r], pix[r]);
    int status[2] = {0, 0};
    float thit[2] = {0.f, 0.f};
    F3 q[2], n[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
        if (live[r]) {   // L2 loads: in the fused kernel the records were written by other SMs
            const float4* hp = reinterpret_cast<const float4*>(L.hits + pix[r]);
            a = __ldcg(hp);
            b = __ldcg(hp + 1);
        }
        q[r] = f3(a.x, a.y, a.z);
        thit[r] = a.w;
        n[r] = f3(b.x, b.y, b.z);
        status[r] = __float_as_int(b.w);
    }
    const DevLight& Lt = P.lights[l];
    bool want[2];
    float dist2[2];
    F3 x0[2], v0[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const F3 D = f3(Lt.pos[0] - q[r].x, Lt.pos[1] - q[r].y, Lt.pos[2] - q[r].z);
        dist2[r] = D.x * D.x + D.y * D.y + D.z * D.z;
        const float lam = (n[r].x * D.x + n[r].y * D.y + n[r].z * D.z) * rsqrtf(dist2[r]);
        want[r] = live[r] && status[r] == 1 && lam > 0.f;
        x0[r] = v0[r] = f3(0.f, 0.f, 0.f);
        if (want[r]) {
            x0[r] = f3(fmaf(kShadowEps, n[r].x, q[r].x), fmaf(kShadowEps, n[r].y, q[r].y),
                       fmaf(kShadowEps, n[r].z, q[r].z));
            float g[6];
            bool ok;
            metric_at(P, x0[r], g, ok);
            const float n2 = g[0] * D.x * D.x + g[3] * D.y * D.y + g[5] * D.z * D.z +
                             2.f * (g[1] * D.x * D.y + g[2] * D.x * D.z + g[4] * D.y * D.z);
            const float inv = rsqrtf(n2);
            v0[r] = f3(D.x * inv, D.y * inv, D.z * inv);
            want[r] = ok;
        }
    }
    int sst[2], sstp[2];
    march_pair<KIND, NB, kPassShadow, MESH>(P, want[0], want[1], pair_of(x0[0], x0[1]), pair_of(v0[0], v0[1]),
                                us, L, unit, sst, sstp, stg, q[0], q[1], dist2[0], dist2[1]);
    bool vis[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        if (want[r]) us.shadow_steps += (unsigned)sstp[r];   // reference-equivalent steps
        vis[r] = want[r] && sst[r] == 1;
    }
    bool last = true;
    if (nl > 1) {
#pragma unroll
        for (int r = 0; r < 2; ++r)
            if (live[r]) {
                RR_CHECK(pix[r] < L.out_pixels, "visibility index");
                L.vis[pix[r] * (unsigned)nl + l] = vis[r] ? 1 : 0;
            }
        __threadfence();
        __syncwarp();
        unsigned before = 0;
        RR_CHECK(unit < (L.n_units + 1) / 2, "unit counter index");
        if (lane == 0) before = atomicAdd(L.done + unit, 1u);
        before = __shfl_sync(kFull, before, 0);
        RR_CHECK(before < (unsigned)nl, "lights-finished counter overrun");
        last = before == (unsigned)nl - 1u;
        if (last) __threadfence();
    }
    if (!last) return;
    uint32_t rgb[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        rgb[r] = 0u;
        if (live[r]) {
            float contrib = 0.f;
            if (status[r] == 1) {
                for (int k = 0; k < nl; ++k) {
#if RR_CHECKS
                    // debug launches pre-fill the visibility bytes with 0xff:
                    // the last finisher must see every other light's byte
                    RR_CHECK(k == l || __ldcg(L.vis + pix[r] * (unsigned)nl + k) <= 1u,
                             "visibility byte not yet published");
#endif
                    const bool lit = k == l ? vis[r] : __ldcg(L.vis + pix[r] * (unsigned)nl + k) != 0;
                    if (!lit) continue;
                    const DevLight& Lk = P.lights[k];
                    const F3 D = f3(Lk.pos[0] - q[r].x, Lk.pos[1] - q[r].y, Lk.pos[2] - q[r].z);
                    const float d2 = D.x * D.x + D.y * D.y + D.z * D.z;
                    const float lam = (n[r].x * D.x + n[r].y * D.y + n[r].z * D.z) * rsqrtf(d2);
                    contrib = fmaf(Lk.intensity, lam, contrib);
                }
            }
            rgb[r] = shade_rgb(P, status[r], thit[r], q[r], P.ambient + contrib);
        }
    }
    store_pair_rgb(L, unit, lane, rgb, stg);
}

// Ray-pair persistent kernel.  Work items are dispensed by one atomic
// counter:
//   kPassShade  : n_pairs primary units with fused shading (no lights);
//   kPassHits   : n_pairs primary units writing hit records;
//   kPassShadow : n_pairs x n_lights shadow units (after a kPassHits launch);
//   kPassFused  : the two above in ONE launch — primary units first, then the
//                 shadow units; a shadow unit waits (rarely: it was dispensed
//                 n_pairs items later) for its primary unit's ready flag, so
//                 the frame has one tail instead of two and no launch gap.
//                 No deadlock: a flag's producer already holds a running warp
//                 and waits on nothing.
template <int KIND, int NB, int PASS, bool MESH>
__global__ void __launch_bounds__(kThreads, KIND == kBumpsRk23 ? RR_MIN_BLOCKS_X2_RK23
                                               : KIND == kDiffeoChain ? (NB != 0 ? RR_MIN_BLOCKS_X2_CHAIN_STATIC
                                                                                 : RR_MIN_BLOCKS_X2_CHAIN)
                                               : KIND == kDiffeo ? (MESH ? RR_MIN_BLOCKS_X2_TWIST_MESH
                                                                     : RR_MIN_BLOCKS_X2_TWIST)
                                               : NB <= 4 ? RR_MIN_BLOCKS_X2_SMALL
                                               : (PASS == kPassFused ? RR_MIN_BLOCKS_X2_FUSED
                                                  : PASS == kPassShadow ? RR_MIN_BLOCKS_X2_SHADOW
                                                  : PASS == kPassHits ? RR_MIN_BLOCKS_X2_HITS
                                                                      : RR_MIN_BLOCKS_X2))
march2_kernel(const __grid_constant__ DevParams P, const __grid_constant__ DevLaunch L) {
    const int lane = threadIdx.x & 31;
    const unsigned n_pairs = (L.n_units + 1) / 2;
    constexpr bool kShadowWork = PASS == kPassShadow || PASS == kPassFused;
    const int nl = kShadowWork ? P.n_lights : 1;
    const unsigned n_primary = PASS == kPassShadow ? 0u : n_pairs;
    const unsigned n_work = n_primary + (kShadowWork ? n_pairs * (unsigned)nl : 0u);
    auto fetch = [&]() {
        unsigned w = 0;
        if (lane == 0) w = atomicAdd(L.counter, 1u);
        // broadcast through REDUX (a uniform-register result), so that
        // everything derived from the work item — the unified loop's
        // per-item pass switch included — stays on the uniform datapath
        return __reduce_max_sync(kFull, w);
    };
    // Two sequential loops (no if/else between the unit kinds inside one
    // loop body: that made ptxas treat the bump loops as divergent and drop
    // their uniform-datapath constant loads).  The warp whose fetch crosses
    // n_primary carries that item into the shadow loop.
    __shared__ PairStage s_stage[kThreads / 32];
    PairStage* stg = &s_stage[threadIdx.x >> 5];
    if constexpr (RR_X2_HITS_STAGED && (PASS == kPassHits || PASS == kPassFused)) {
        __shared__ float4 s_chord[kThreads / 32][4 * kUnit];
        stg->chord = s_chord[threadIdx.x >> 5];
    }
    unsigned work = fetch();
    if constexpr (PASS != kPassShadow) {
        constexpr int kPrim = PASS == kPassFused ? kPassHits : PASS;
        while (work < n_primary) {
            // expensive units first (L.order: the previous frame's costs,
            // sorted on the device); outputs do not depend on the order
            const unsigned unit = L.order ? __ldg(L.order + work) : work;
            UnitStats us{};
            pair_primary<KIND, NB, kPrim, MESH>(P, L, unit, lane, us, stg);
            if (L.unit_cost && lane == 0)                       // warp-loop iterations of the unit
                L.unit_cost[unit] = (unsigned short)min(us.cnt.lane_slots / 2u, 65535u);
            if constexpr (PASS == kPassFused) {                 // publish the hit records
                __threadfence();
                __syncwarp();
                if (lane == 0) atomicExch(L.ready + unit, 1u);
            }
            flush_unit_stats(L, us, lane, false);
            work = fetch();
        }
    }
    if constexpr (kShadowWork) {
        while (work < n_work) {
            const unsigned w = work - n_primary;
            const unsigned unit = L.order2 ? __ldg(L.order2 + w / (unsigned)nl) : w / (unsigned)nl;
            if constexpr (PASS == kPassFused) {
                RR_CHECK(unit < n_pairs, "ready flag index");
                // whole-warp polling of the unit's ready flag (dispensed
                // n_pairs items after its primary unit: normally already set)
                for (;;) {
                    unsigned f = 0;
                    if (lane == 0) f = atomicAdd(L.ready + unit, 0u);
                    if (__shfl_sync(kFull, f, 0)) break;
                    __nanosleep(256);
                }
                __threadfence();
            }
            UnitStats us{};
            pair_shadow<KIND, NB, MESH>(P, L, unit, (int)(w % (unsigned)nl), nl, lane, us, stg);
            if (L.unit_cost2 && lane == 0)                      // max over the unit's lights
                atomicMax(L.unit_cost2 + unit, min(us.cnt.lane_slots / 2u, 65535u));
            flush_unit_stats(L, us, lane, true);
            work = fetch();
        }
    }
    if (L.mode == kModeFrame && L.n_shards > 1) __threadfence_system();
}

template <int KIND, int NB, int SCHEME, int PASS, bool MESH>
int occupancy_of() {
    static int occ = [] {
        int n = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, march_kernel<KIND, NB, SCHEME, PASS, MESH>,
                                                      kThreads, 0);
        return n > 0 ? n : 1;
    }();
    return occ;
}

template <int KIND, int NB, int SCHEME, int PASS, bool MESH>
cudaError_t launch_pass(const DevParams& P, const DevLaunch& L, cudaStream_t s, int num_sms) {
    const unsigned warps_needed = L.n_units;
    unsigned blocks = (unsigned)(num_sms * occupancy_of<KIND, NB, SCHEME, PASS, MESH>());
    const unsigned max_useful = (warps_needed + 3) / 4;
    if (blocks > max_useful) blocks = max_useful;
    if (blocks == 0) blocks = 1;
    march_kernel<KIND, NB, SCHEME, PASS, MESH><<<blocks, kThreads, 0, s>>>(P, L);
    return cudaGetLastError();
}

template <int KIND, int NB, int PASS, bool MESH>
int occupancy_of2() {
    static int occ = [] {
        int n = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, march2_kernel<KIND, NB, PASS, MESH>, kThreads, 0);
        return n > 0 ? n : 1;
    }();
    return occ;
}

template <int KIND, int NB, int PASS, bool MESH>
cudaError_t launch_pass2(const DevParams& P, const DevLaunch& L, cudaStream_t s, int num_sms) {
    const unsigned warps_needed = (L.n_units + 1) / 2;
    const int occ = occupancy_of2<KIND, NB, PASS, MESH>();
    unsigned blocks = (unsigned)(num_sms * occ);
#if RR_SMALL_LAUNCH_CTAS
    // Launches with few work items per SM (a 1080p frame split over 4 or 8
    // GPUs) end on their slowest units, which run faster with fewer
    // co-resident warps: 2 + items/18 CTAs per SM below the full occupancy
    // (C3 shards at N = 8: 1.96 -> 1.55 ms, N = 4: 2.81 -> 2.57 ms; full
    // frames keep the full grid: profiles/r2z_small_launch_ab.log)
    {
        const double items = (double)warps_needed * (PASS == kPassShadow ? (double)P.n_lights : 1.0);
        const double per_sm = items / num_sms;
        if (per_sm < 18.0 * (occ - 2)) {
            const int want = (int)lround(2.0 + per_sm / 18.0);
            const int ctas = want < 2 ? 2 : (want > occ ? occ : want);
            blocks = (unsigned)(num_sms * ctas);
        }
    }
#endif
    const unsigned max_useful = (warps_needed + 3) / 4;
    if (blocks > max_useful) blocks = max_useful;
    if (blocks == 0) blocks = 1;
    march2_kernel<KIND, NB, PASS, MESH><<<blocks, kThreads, 0, s>>>(P, L);
    return cudaGetLastError();
}

template <int KIND, int NB, bool MESH>
cudaError_t launch_variant2(const DevParams& P, const DevLaunch& L, cudaStream_t s, int num_sms) {
    if (P.n_lights == 0 || L.mode == kModeRays) return launch_pass2<KIND, NB, kPassShade, MESH>(P, L, s, num_sms);
#if RR_X2_FUSED
    return launch_pass2<KIND, NB, kPassFused, MESH>(P, L, s, num_sms);
#endif
    cudaError_t e = launch_pass2<KIND, NB, kPassHits, MESH>(P, L, s, num_sms);
    if (e != cudaSuccess) return e;
    DevLaunch L2 = L;
    L2.counter = L.counter + 1;
    L2.lpp = 1;
    return launch_pass2<KIND, NB, kPassShadow, MESH>(P, L2, s, num_sms);
}

// Without lights: one fused launch.  With lights (EXTENSION): a hit-record
// pass and a shadow+shade pass over the same units (each with its own unit
// counter: L.counter[0] and L.counter[1]).  Scenes with meshes use the MESH
// variants (BVH traversal compiled in; kept out of the mesh-free kernels).
template <int KIND, int NB, int SCHEME, bool MESH>
cudaError_t launch_variant(const DevParams& P, const DevLaunch& L, cudaStream_t s, int num_sms) {
    if (P.n_lights == 0 || L.mode == kModeRays)
        return launch_pass<KIND, NB, SCHEME, kPassShade, MESH>(P, L, s, num_sms);
    cudaError_t e = launch_pass<KIND, NB, SCHEME, kPassHits, MESH>(P, L, s, num_sms);
    if (e != cudaSuccess) return e;
    DevLaunch L2 = L;
    L2.counter = L.counter + 1;
    // lights per pixel marched in one unit: 1.  Pairing 2 lights x 16 pixels per
    // warp was measured slower on C3 (27.2 vs 23.7 ms/frame): two light
    // directions in one warp widen the culling union and split coherence.
    L2.lpp = 1;
    L2.n_units = L.n_units * L2.lpp;
    return launch_pass<KIND, NB, SCHEME, kPassShadow, MESH>(P, L2, s, num_sms);
}

} // namespace
} // namespace rr
