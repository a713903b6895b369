// common.cuh -- shared device helpers for the B200 FT-SZ kernels (sm_100a).
//
// Exact-arithmetic helpers: the reference evaluates every per-point formula in float64 with
// a fixed operand order and float32 storage.  All float64 math
// here uses __dadd_rn/__dmul_rn (never contracted to DFMA) and the file is compiled with
// -fmad=false.  Measured on B200 (tools/fp64_probe.cu): DADD/DMUL issue at 2 warp-ops/clk/SM,
// F2F / F2I / I2F at ~1/4 of that and DDIV at 1/14, so conversions and divisions are replaced
// by exact integer bit manipulations wherever the result is provably identical.
#pragma once
#include <type_traits>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/ftlz_b200.h"

#define FTLZ_DEV __device__ __forceinline__

typedef unsigned long long u64;
typedef uint32_t u32;
typedef uint16_t u16;
typedef uint8_t u8;

// ------------------------------------------------------------------------------------------
// device status: first error wins (kernels no-op once code != 0)
struct DevStatus {
    int code;
    int kind;
    long long offset, block, a, b;
    long long order;          // ordering key for "first error" selection
    int lock;
    int pad;
};

FTLZ_DEV void dev_fail(DevStatus* st, int code, int kind, long long offset, long long block,
                       long long a, long long b, long long order) {
    // keep the error with the smallest `order` (sequential reference semantics)
    while (atomicCAS(&st->lock, 0, 1) != 0) {
    }
    __threadfence();
    volatile DevStatus* vs = st;
    if (vs->code == 0 || order < vs->order) {
        vs->code = code;
        vs->kind = kind;
        vs->offset = offset;
        vs->block = block;
        vs->a = a;
        vs->b = b;
        vs->order = order;
    }
    __threadfence();
    atomicExch(&st->lock, 0);
}

FTLZ_DEV bool dev_failed(const DevStatus* st) { return *(volatile const int*)&st->code != 0; }

// ------------------------------------------------------------------------------------------
// exact conversions without the conversion pipe

// float32 -> float64, exact (IEEE widening).  Normal and zero inputs use integer ops only;
// subnormal / inf / NaN fall back to F2F (identical result; rare).
FTLZ_DEV double f32_to_f64(float f) {
    u32 u = __float_as_uint(f);
    u32 e = (u >> 23) & 0xffu;
    if (e == 0u || e == 0xffu) {
        if ((u & 0x7fffffffu) == 0u) return __hiloint2double((int)(u & 0x80000000u), 0);
        return (double)f;
    }
    u32 hi = (u & 0x80000000u) | ((e + 896u) << 20) | ((u >> 3) & 0xfffffu);
    u32 lo = u << 29;
    return __hiloint2double((int)hi, (int)lo);
}

// integer -> float64, exact (one I2F.F64: a single issue slot on the conversion pipe, where the
// 2^52-magic form took three)
FTLZ_DEV double int_to_f64(int n) { return __int2double_rn(n); }

FTLZ_DEV u64 dbits(double d) { return (u64)__double_as_longlong(d); }

// exact u32 division by a launch-constant divisor: q = hi64(n * ceil(2^64 / d)), which is
// floor(n / d) for every n, d < 2^32 (error < n / 2^64 < 1/d); d == 1 is passed through.
struct FastDiv {
    u64 m;
    u32 d;
    u32 pad;
};
FTLZ_DEV u32 fdiv(u32 n, const FastDiv& f) { return f.d == 1u ? n : (u32)__umul64hi((u64)n, f.m); }
static inline FastDiv make_fastdiv(u32 d) {
    FastDiv f;
    f.d = d;
    f.m = d <= 1u ? 0ull : (~0ull / d) + 1ull;
    f.pad = 0;
    return f;
}

// ordered-int encoding of float32 for atomic min/max (NaN handled separately)
FTLZ_DEV u32 f2ord(float f) {
    u32 u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
FTLZ_DEV float ord2f(u32 o) {
    u32 u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
    return __uint_as_float(u);
}

// ------------------------------------------------------------------------------------------
// quantizer (pipeline.py:271-279 == quantize.py:37-52), exact.
//   h = |diff| / (2 eb); small = h <= 2*cap; q = floor(fl((small ? h : 0) + 0.5)); sign;
//   b = center + q; ok = small && 1 <= b <= cap-1.
// Fast path: h' = |diff| * rcp (rcp = RN(1/(2eb))), |h' - h| <= 2 ulp.  The decision
// floor(fl(h+0.5)) / (h <= 2cap) can only differ when h' lies within a few ulps of a
// threshold; those points (probability ~2^-40) take the exact IEEE division.
struct QuantParams {
    double eb, twoeb, rcp;  // rcp = 1/(2eb) rounded; exact_div != 0 forces DDIV
    double capd2;           // 2.0 * cap
    u64 capd2_bits;
    u64 eb_bits;
    int cap, center;
    int exact_div;
    int pad;
    double twoeb_dup;       // second copy of 2*eb: the duplicated evaluation loads its own operand
    // float32 decision path (quant_reg10.cu)
    float rcp32, eb32;      // RN32(1 / (2 eb)), RN32(eb)
    float band32, sbig;     // guard band around eb (eb32 * 2^-20); |s| >= sbig -> unpredictable
    int fast32;             // 0: every point takes the reference formulation
    int pad2;
};

// floor(t) for t in [0, 2^31): integer extraction from the bit pattern
FTLZ_DEV int floor_pos(double t, int* near_int) {
    u64 b = dbits(t);
    int E = (int)(b >> 52) - 1023;
    if (E < 0) {
        // t < 1: floor 0; near 1 from below?
        *near_int = (E == -1) && ((b & 0xfffffffffffffull) > 0xfffffffffff00ull);
        return 0;
    }
    u64 m = (b & 0xfffffffffffffull) | 0x10000000000000ull;
    int sh = 52 - E;
    u64 fracmask = (sh >= 64) ? ~0ull : ((1ull << sh) - 1ull);
    u64 frac = m & fracmask;
    // within 64 ulp of an integer (either side)
    *near_int = ((frac + 64ull) & fracmask) < 128ull;
    return (int)(m >> sh);
}

// returns the bin (0 = unpredictable); *ok as the reference's `ok` mask
FTLZ_DEV int quantize(const QuantParams& Q, double diff, bool* ok) {
    double ad = fabs(diff);
    bool small;
    int q;
    bool slow = Q.exact_div != 0;
    if (!slow) {
        double h = __dmul_rn(ad, Q.rcp);
        u64 hb = dbits(h);
        // small decision: exact unless h' within 2^-40 relative of 2*cap
        small = hb <= Q.capd2_bits;
        u64 d = hb > Q.capd2_bits ? hb - Q.capd2_bits : Q.capd2_bits - hb;
        if (d < 4096ull) slow = true;
        if (!slow) {
            double t = __dadd_rn(small ? h : 0.0, 0.5);
            int near_int;
            q = floor_pos(t, &near_int);
            if (near_int && small) slow = true;
        }
    }
    if (slow) {
        double h = __ddiv_rn(ad, Q.twoeb);
        small = h <= Q.capd2;
        double t = __dadd_rn(small ? h : 0.0, 0.5);
        q = (int)floor(t);
    }
    if (diff < 0.0) q = -q;
    int b = Q.center + q;
    *ok = small && b >= 1 && b <= Q.cap - 1;
    return *ok ? b : 0;
}

// |x - y| <= eb for non-negative comparisons via bit patterns (NaN -> false)
FTLZ_DEV bool within_eb(double diff_abs_src, u64 eb_bits) {
    u64 b = dbits(diff_abs_src) & 0x7fffffffffffffffull;
    return b <= eb_bits;
}

// ------------------------------------------------------------------------------------------
// opaque copy: forces a genuine second evaluation for duplicated evaluation (pipeline.py:157-179)
FTLZ_DEV double opaque(double x) {
    double y;
    asm volatile("mov.b64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}

// ------------------------------------------------------------------------------------------
// warp reductions
FTLZ_DEV u64 warp_sum_u64(u64 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
FTLZ_DEV unsigned warp_sum_u32(unsigned v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// u64 warp sum through three 22-bit limbs and REDUX (each limb sum < 2^27)
FTLZ_DEV u64 warp_sum_u64_redux(u64 v) {
    const u32 l0 = (u32)v & 0x3fffffu, l1 = (u32)(v >> 22) & 0x3fffffu, l2 = (u32)(v >> 44);
    const u64 s0 = __reduce_add_sync(0xffffffffu, l0), s1 = __reduce_add_sync(0xffffffffu, l1),
              s2 = __reduce_add_sync(0xffffffffu, l2);
    return s0 + (s1 << 22) + (s2 << 44);
}

// ------------------------------------------------------------------------------------------
// geometry (core.py:113-157)
struct Geom {
    long long nx, ny, nz;
    long long cx, cy, cz, nb;
    int e;
    int rx, ry, rz;     // trailing extents (== e when the axis divides)
    int vmax;           // e^3
    int nvmax8;         // vmax rounded up to a multiple of 8 (bins layout)
    FastDiv fcz, fcy;   // divisors for block coordinates (used when nb < 2^32)
};

FTLZ_DEV void block_coords(const Geom& g, long long b, long long* bi, long long* bj, long long* bk) {
    if (g.nb < (1ll << 32)) {
        u32 t = fdiv((u32)b, g.fcz);
        *bk = (long long)((u32)b - t * (u32)g.cz);
        u32 i = fdiv(t, g.fcy);
        *bi = i;
        *bj = (long long)(t - i * (u32)g.cy);
        return;
    }
    long long t = b / g.cz;
    *bk = b - t * g.cz;
    *bi = t / g.cy;
    *bj = t - *bi * g.cy;
}

FTLZ_DEV int extent_id(const Geom& g, long long bi, long long bj, long long bk) {
    return ((bi == g.cx - 1 && g.rx != g.e) ? 4 : 0) | ((bj == g.cy - 1 && g.ry != g.e) ? 2 : 0) |
           ((bk == g.cz - 1 && g.rz != g.e) ? 1 : 0);
}

FTLZ_DEV void extent_of(const Geom& g, int xid, int* bx, int* by, int* bz) {
    *bx = (xid & 4) ? g.rx : g.e;
    *by = (xid & 2) ? g.ry : g.e;
    *bz = (xid & 1) ? g.rz : g.e;
}

// bins layout shared by the quantizer (writer) and the encoder (reader): block-contiguous,
// nvmax8 u16 per block (16-byte aligned rows)
FTLZ_DEV size_t bins_index(const Geom& g, long long b, int p) { return (size_t)b * (size_t)g.nvmax8 + (size_t)p; }

struct BlockInfo {
    long long b, bi, bj, bk;
    int xid, bx, by, bz, vol;
    bool valid;
};

FTLZ_DEV BlockInfo block_info(const Geom& g, long long b) {
    BlockInfo B;
    B.b = b;
    B.valid = b < g.nb;
    if (!B.valid) b = g.nb - 1;
    block_coords(g, b, &B.bi, &B.bj, &B.bk);
    B.xid = extent_id(g, B.bi, B.bj, B.bk);
    extent_of(g, B.xid, &B.bx, &B.by, &B.bz);
    B.vol = B.bx * B.by * B.bz;
    return B;
}

// per-extent plans (pairwise-sum leaves, wavefront order, coordinates) built on the host
struct ExtPlan {
    int bx, by, bz, vol;
    int nleaf, leaf_off;     // leaves of the pairwise tree over vol elements
    int ns, nsleaf, sleaf_off;  // samples (SAMPLE_STRIDE=8) and their pairwise leaves
    int coord_off;           // vol u32 entries: i | j<<8 | k<<16 (row-major p -> coords)
    int wave_off;            // vol u16-in-u32 entries: p ordered by plane i+j+k
    int plane_off;           // (bx+by+bz-1) u32 plane start offsets (+1 sentinel)
    int nplanes;
    int exl;                 // ceil(log2(2 (max edge - 1) vol)): exact-sum condition of k_prep
    double den[3];           // regression denominators vol * (n^2 - 1) / 12.0 per axis (predict.py:98)
};

// leaf descriptor: start (elements), len, combine count after pushing this leaf
struct Leaf {
    int start;
    int len;
    int ncomb;
    int pad;
};

// block-wide bitonic sort of n_pow2 u64 keys (ascending); all threads of the CTA participate
// Bitonic sort of n_pow2 keys in shared memory by the whole CTA (blockDim a multiple of 32).
// Element e = tid + r * blockDim lives in register r of thread tid while in registers: the
// stages with j < 32 run as warp shuffles and those with j >= blockDim inside one thread, so
// only 32 <= j < blockDim need shared memory and a barrier (42 barriers at 8192 keys and
// 1024 threads instead of 91).  Same comparisons and result as the plain network.
#define BS_MAXR 8
FTLZ_DEV void bitonic_sort_u64_plain(u64* keys, int n_pow2);
FTLZ_DEV void bitonic_sort_u64(u64* keys, int n_pow2) {
    const int T = blockDim.x, tid = threadIdx.x, lane = tid & 31;
    const int R = (n_pow2 + T - 1) / T;
    if (R > BS_MAXR || (T & 31) || (T & (T - 1)) || n_pow2 < 64) {
        bitonic_sort_u64_plain(keys, n_pow2);
        return;
    }
    u64 v[BS_MAXR];
    auto load = [&]() {
#pragma unroll
        for (int r = 0; r < BS_MAXR; r++)
            if (r < R && tid + r * T < n_pow2) v[r] = keys[tid + r * T];
    };
    auto store = [&]() {
#pragma unroll
        for (int r = 0; r < BS_MAXR; r++)
            if (r < R && tid + r * T < n_pow2) keys[tid + r * T] = v[r];
        __syncthreads();
    };
    // stages j < 32 of merge size k (k >= 2): partner e ^ j is lane ^ j of the same register
    auto warp_stages = [&](int k) {
        for (int j = min(k >> 1, 16); j > 0; j >>= 1) {
#pragma unroll
            for (int r = 0; r < BS_MAXR; r++) {
                if (r >= R) break;
                const int e = tid + r * T;
                const u64 o = __shfl_xor_sync(0xffffffffu, v[r], j);
                const bool up = (e & k) == 0, lower = (e & j) == 0;
                const u64 mn = v[r] < o ? v[r] : o, mx = v[r] < o ? o : v[r];
                v[r] = (lower == up) ? mn : mx;
            }
        }
    };
    load();
    for (int k = 2; k <= 32 && k <= n_pow2; k <<= 1) warp_stages(k);
    store();
    for (int k = 64; k <= n_pow2; k <<= 1) {
        int j = k >> 1;
        if (j >= T) {
            // partner in another register of the same thread
            load();
            // register distance rj = j / T in {4, 2, 1}: compile-time indices keep v in registers
            auto reg_stage = [&](auto rjc) {
                constexpr int RJ = decltype(rjc)::value;
#pragma unroll
                for (int r = 0; r < BS_MAXR; r++) {
                    if ((r & RJ) || r + RJ >= BS_MAXR) continue;
                    if (r + RJ >= R) continue;
                    const int e = tid + r * T;
                    const bool up = (e & k) == 0;
                    const u64 a = v[r], c = v[r + RJ];
                    const bool sw = (a > c) == up;
                    v[r] = sw ? c : a;
                    v[r + RJ] = sw ? a : c;
                }
            };
            for (; j >= T; j >>= 1) {
                const int rj = j / T;
                if (rj == 4) reg_stage(std::integral_constant<int, 4>());
                else if (rj == 2) reg_stage(std::integral_constant<int, 2>());
                else reg_stage(std::integral_constant<int, 1>());
            }
            store();
        }
        for (; j >= 32; j >>= 1) {
            for (int i = tid; i < n_pow2; i += T) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const u64 a = keys[i], c = keys[ixj];
                    const bool up = (i & k) == 0;
                    if ((a > c) == up) { keys[i] = c; keys[ixj] = a; }
                }
            }
            __syncthreads();
        }
        load();
        warp_stages(k);
        store();
    }
}

FTLZ_DEV void bitonic_sort_u64_plain(u64* keys, int n_pow2) {
    for (int k = 2; k <= n_pow2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n_pow2; i += blockDim.x) {
                int ixj = i ^ j;
                if (ixj > i) {
                    u64 a = keys[i], c = keys[ixj];
                    bool up = (i & k) == 0;
                    if ((a > c) == up) { keys[i] = c; keys[ixj] = a; }
                }
            }
            __syncthreads();
        }
    }
}


// ------------------------------------------------------------------------------------------
#define HWIN 4096   // shared-memory histogram window around the quantizer center

// histogram increment: shared window (flushed once per CTA) or global for outliers
FTLZ_DEV void hist_add(u32* hwin, u64* ghist, int wlo, int bin, u32 cnt) {
    unsigned o = (unsigned)(bin - wlo);
    if (o < HWIN) atomicAdd(&hwin[o], cnt);
    else atomicAdd(&ghist[bin], (u64)cnt);
}

FTLZ_DEV void hist_flush(u32* hwin, u64* ghist, int wlo, int cap) {
    for (int t = threadIdx.x; t < HWIN; t += blockDim.x) {
        u32 v = hwin[t];
        int s = wlo + t;
        if (v && s >= 0 && s < cap) atomicAdd(&ghist[s], (u64)v);
    }
}

