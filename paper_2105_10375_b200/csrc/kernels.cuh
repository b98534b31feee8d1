// kernels.cuh -- the DCP head's non-GEMM kernels (hot-path steps a1, a3, a6, a8,
// a9 and a10 of DESIGN.md section 2).  All of them are HBM- or latency-bound.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "dcp_main.cuh"
#include "dcp_pc.cuh"
#include "sm100.cuh"

namespace f2c {

enum : int { ERR_OK = 0, ERR_PAIRING = 4, ERR_DEVICE = 7 };
// detail codes kept next to the status (scal->err_detail) for f2c_last_error
enum : int {
    DET_NONE = 0, DET_BAD_LABEL = 1, DET_ZERO_ROW = 2, DET_PAIRING = 3, DET_NONFINITE = 4,
    DET_UNDERFLOW = 5, DET_DUP_BLOCK = 6
};

struct Scalars {          // lives at the start of the per-rank scratch
    int err;              // latched f2c_status
    int err_detail;       // DET_*
    int tmax_bits;        // max ||T_c|| over rows ever written (float bits, >= 0)
    int n_pos;            // in-pool rows of the last loss call
    int n_neg;
    int neg0;             // first compacted out-of-pool row (NEXT-3 hinge / max): n_pos rounded
                          // up to a warp (32 rows), so no warp mixes softmax rows and cosine rows
    int n_rows;           // compacted rows the main kernel processes (n_pos, or neg0 + N_neg
                          // when the out-of-pool rows go through it: NEXT-3 hinge / max)
    double loss3[3];      // L, L_ce, L_cos (fp64) of the last loss call
    unsigned long long n_pos_sum;  // sum of n_pos over loss calls (bench accounting)
    long long n_app;      // rows appended by the last refresh-in-place enqueue (NEXT-3)
    unsigned loss_done;   // CTAs of the final per-row kernel done (the last one sums the loss)
    int refine;           // R1 fallback: some row's reference was lowered, re-run the fused kernel
    int S_sched;          // dcp_pc_kernel's range count for this loss call (k_compact)
    int *err_mirror;      // mapped pinned host words {err, detail} of this shard: the host reads
                          // them at the next call on the handle without synchronising
};

__device__ __forceinline__ void latch(Scalars *s, int code, int detail) {
    if (atomicCAS(&s->err, 0, code) == 0) {
        s->err_detail = detail;
        if (s->err_mirror) {  // (rare: one system-scope store pair per latched error)
            volatile int *m = s->err_mirror;
            m[1] = detail;
            __threadfence_system();
            m[0] = code;
            __threadfence_system();
        }
    }
}

__device__ __forceinline__ uint64_t hash64(uint64_t z) {
    z ^= z >> 33;
    z *= 0xff51afd7ed558ccdull;
    z ^= z >> 33;
    z *= 0xc4ceb9fe1a85ec53ull;
    z ^= z >> 33;
    return z;
}

// ------------------------------------------------------------------ a3: the shard's label index
// label -> newest write index (seq) of the label among this shard's slots, or -1 once that slot
// has been overwritten.  Older copies of a label are overwritten before its newest one (ring
// order; a refresh-in-place keeps a slot's seq), so value -1 means the label has left the shard,
// and target resolution (D8) is one lookup per batch row instead of a pass over the pool labels.
// The enqueue kernels update it for every appended row: evict (old label, old seq) with a CAS
// that only succeeds if that seq is still the label's newest, then insert (label, new seq) with
// atomicMax -- the two commute, so rows of one block may update the same label in any order.
// Open addressing with linear probing over HI (a power of two) entries; keys are never removed,
// and the host rebuilds the table from the shard's labels (k_idx_build) before the key count can
// exceed HI / 2.
struct LabelIndex {
    int64_t *keys;   // [HI], -1 = empty
    long long *vals; // [HI], newest seq or -1
    int HI;
};
__device__ __forceinline__ int idx_find(const LabelIndex &ix, int64_t key) {
    unsigned h = static_cast<unsigned>(hash64(static_cast<uint64_t>(key))) & (ix.HI - 1);
    for (;;) {
        const int64_t k = ix.keys[h];
        if (k == key) return static_cast<int>(h);
        if (k == -1) return -1;
        h = (h + 1) & (ix.HI - 1);
    }
}
__device__ __forceinline__ int idx_claim(const LabelIndex &ix, int64_t key) {
    unsigned h = static_cast<unsigned>(hash64(static_cast<uint64_t>(key))) & (ix.HI - 1);
    for (;;) {
        const unsigned long long old = atomicCAS(reinterpret_cast<unsigned long long *>(ix.keys + h),
                                                 static_cast<unsigned long long>(-1ll), static_cast<unsigned long long>(key));
        if (old == static_cast<unsigned long long>(-1ll) || old == static_cast<unsigned long long>(key))
            return static_cast<int>(h);
        h = (h + 1) & (ix.HI - 1);
    }
}
__device__ __forceinline__ void idx_evict(const LabelIndex &ix, int64_t key, long long seq) {
    const int h = idx_find(ix, key);
    if (h >= 0) atomicCAS(reinterpret_cast<unsigned long long *>(ix.vals + h), static_cast<unsigned long long>(seq),
                          static_cast<unsigned long long>(-1ll));
}
__device__ __forceinline__ void idx_insert(const LabelIndex &ix, int64_t key, long long seq) {
    atomicMax(ix.vals + idx_claim(ix, key), seq);
}
__device__ __forceinline__ long long idx_lookup(const LabelIndex &ix, int64_t key) {
    const int h = idx_find(ix, key);
    return h < 0 ? -1ll : ix.vals[h];
}
// slot of block row j: (E + j) mod C with e0 = E mod C (j < m_glob <= C, so one conditional
// subtract: a 64-bit modulo per row and lane cost more than the row copy itself), or the planned
// write index of a refresh-in-place enqueue
__device__ __forceinline__ int64_t enq_slot(int64_t j, int64_t e0, int64_t C, const int64_t *__restrict__ dst_seq) {
    if (dst_seq) return dst_seq[j] % C;
    const int64_t c = e0 + j;
    return c >= C ? c - C : c;
}

// The label pass of an enqueue (one THREAD per block row, so the index's dependent DRAM round
// trips of all rows overlap; the feature copy runs in separate warp-per-row loops that never touch
// the labels): the row is written at seq qn -- pure Eq. 7 appends every row, a refresh-in-place
// enqueue (dst_seq) only the rows with qn >= E (a refreshed row keeps its label and seq).  Evict
// the slot's previous label (content qn - C, when qn >= C) if that seq is still its newest, insert
// the new label, write the slot's label.
__device__ __forceinline__ void enqueue_labels(const int64_t *__restrict__ y, int64_t m_glob, int64_t E, int64_t C,
                                               int64_t lo, int64_t hi, int64_t *__restrict__ lab,
                                               const int64_t *__restrict__ dst_seq, const LabelIndex &ix) {
    const int64_t e0 = E % C;
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < m_glob;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t qn = dst_seq ? dst_seq[j] : E + j;
        const int64_t c = enq_slot(j, e0, C, dst_seq);
        if (c < lo || c >= hi) continue;
        const int64_t yl = y[j];
        if (yl < 0) continue;  // (latched by the copy loop)
        if (ix.keys != nullptr && qn >= E) {
            const int64_t yo = lab[c - lo];
            if (qn >= C && yo >= 0) idx_evict(ix, yo, qn - C);
            idx_insert(ix, yl, qn);
        }
        lab[c - lo] = yl;
    }
}

__global__ void k_idx_clear(LabelIndex ix) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ix.HI; i += gridDim.x * blockDim.x) {
        ix.keys[i] = -1;
        ix.vals[i] = -1;
    }
}
// (re)build from the shard's occupied slots [0, n_occ_loc): seq(c) = c + C floor((E-1-c) / C)
__global__ void k_idx_build(LabelIndex ix, const int64_t *__restrict__ lab, int64_t n_occ_loc, int64_t lo, int64_t C,
                            int64_t E) {
    for (int64_t cl = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; cl < n_occ_loc;
         cl += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t L = lab[cl];
        if (L < 0) continue;
        const int64_t c = lo + cl;
        idx_insert(ix, L, c + C * ((E - 1 - c) / C));
    }
}
// newest local seq of each of n labels (-1: not in this shard)
__global__ void k_idx_lookup(LabelIndex ix, const int64_t *__restrict__ y, int64_t n, int64_t *__restrict__ seq) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t key = y[i];
    seq[i] = key < 0 ? -1 : idx_lookup(ix, key);
}

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }

template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }

// ------------------------------------------------------------------ a1: enqueue
// The pool sum mu = sum over occupied slots of w_c T_bar_c (w_c = 1 for K = 1; reading R3) of
// the L_cos gradient is kept per shard in 64-bit fixed point (quantum 2^-36): every slot's
// contribution is rounded once, the same way whenever it is added or removed, and integer
// addition is exact and associative, so the running sum equals the sum over the current pool
// exactly (any order, any number of steps).  The enqueue kernels read each overwritten row
// before storing the new one and add (new - old) contributions to a per-warp sum in shared
// memory (lanes own distinct columns: plain adds), then one global atomic per column per
// block; set_state rebuilds it (k_mu_sum).
constexpr float MU_FX_SCALE = 68719476736.0f;  // 2^36
constexpr double MU_FX_INV = 1.0 / 68719476736.0;
__device__ __forceinline__ long long mu_fx_of(float v) { return __float2ll_rn(v * MU_FX_SCALE); }
constexpr int MU_WARPS = 8;  // (256-thread enqueue blocks)
__device__ __forceinline__ void mu_block_init(long long (*smu)[512], int d) {
    for (int i = threadIdx.x; i < MU_WARPS * 512; i += blockDim.x) smu[i / 512][i % 512] = 0;
    __syncthreads();
}
__device__ __forceinline__ void mu_block_flush(const long long (*smu)[512], int d, unsigned long long *mu_fx) {
    __syncthreads();
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        long long v = 0;
#pragma unroll
        for (int w = 0; w < MU_WARPS; ++w) v += smu[w][i];
        if (v) atomicAdd(mu_fx + i, static_cast<unsigned long long>(v));
    }
}
// Eq. 7 / Algorithm 1: global block row j -> slot (E+j) mod C.
// One warp per block row; the rows owned by this shard [lo, hi) are copied with
// 16-byte vector loads/stores (bit-exact; labels and the label index: enqueue_labels), and the running
// max row norm (the softmax reference bound) updated.
__global__ void __launch_bounds__(256) k_enqueue(const uint8_t *__restrict__ g, const int64_t *__restrict__ y,
                                                 int64_t m_glob, int64_t E, int64_t C, int64_t lo, int64_t hi,
                                                 int row_bytes, int dtype, uint8_t *__restrict__ T,
                                                 int64_t *__restrict__ lab, Scalars *sc,
                                                 const int64_t *__restrict__ dst_seq,
                                                 unsigned long long *__restrict__ mu_fx, LabelIndex ix,
                                                 __nv_bfloat16 *__restrict__ Tsh) {
    __shared__ float wmax[8];
    __shared__ long long smu[MU_WARPS][512];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    const int epv = dtype == 0 ? 8 : 4;  // elements per 16-byte vector
    enqueue_labels(y, m_glob, E, C, lo, hi, lab, dst_seq, ix);
    mu_block_init(smu, (row_bytes / 16) * epv);  // d columns
    // the lane's mu partial in registers: a lane owns the same <= 16 columns of every row it copies
    // (per-element smem updates were 16-way bank-conflicted and bounded the kernel)
    long long acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0;
    const int nvec = row_bytes / 16;
    float nmax = 0.f;
    const int64_t e0 = E % C;
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + wib; j < m_glob; j += nwarps) {
        // pure Eq. 7: row j -> slot (E + j) mod C; refresh-in-place (NEXT-3): the planned slot
        const int64_t c = enq_slot(j, e0, C, dst_seq);
        if (c < lo || c >= hi) continue;
        const int64_t yl = y[j];
        if (yl < 0) {
            if (lane == 0) latch(sc, ERR_DEVICE, DET_BAD_LABEL);
            continue;
        }
        const int4 *src = reinterpret_cast<const int4 *>(g + j * row_bytes);
        int4 *dst = reinterpret_cast<int4 *>(T + (c - lo) * row_bytes);
        float ss = 0.f;
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {  // 2 independent 16-B loads in flight per lane
            const int u0 = h2 * 64;
            if (u0 >= nvec) break;
            int4 v[2], ov[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int u = u0 + q * 32 + lane;
                if (u < nvec) {
                    v[q] = __ldcs(src + u);
                    ov[q] = dst[u];  // the overwritten row (its mu contribution leaves)
                }
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int u = u0 + q * 32 + lane;
                if (u >= nvec) continue;
                __stcs(dst + u, v[q]);
                const uint32_t w[4] = {static_cast<uint32_t>(v[q].x), static_cast<uint32_t>(v[q].y),
                                       static_cast<uint32_t>(v[q].z), static_cast<uint32_t>(v[q].w)};
                const uint32_t o[4] = {static_cast<uint32_t>(ov[q].x), static_cast<uint32_t>(ov[q].y),
                                       static_cast<uint32_t>(ov[q].z), static_cast<uint32_t>(ov[q].w)};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if (dtype == 0) {
                        const float a = __uint_as_float(w[i] << 16), b = __uint_as_float(w[i] & 0xffff0000u);
                        ss += a * a + b * b;
                        const float oa = __uint_as_float(o[i] << 16), ob = __uint_as_float(o[i] & 0xffff0000u);
                        acc[(q * 8 + 2 * i) & 15] += mu_fx_of(a) - mu_fx_of(oa);
                        acc[(q * 8 + 2 * i + 1) & 15] += mu_fx_of(b) - mu_fx_of(ob);
                    } else {
                        const float a = __uint_as_float(w[i]);
                        ss += a * a;
                        acc[h2 * 8 + q * 4 + i] += mu_fx_of(a) - mu_fx_of(__uint_as_float(o[i]));
                    }
                }
                if (dtype != 0 && Tsh) {  // fp32 pool: its bf16 shadow (the P x pool GEMM's operand)
                    const __nv_bfloat162 s0 = __floats2bfloat162_rn(__uint_as_float(w[0]), __uint_as_float(w[1]));
                    const __nv_bfloat162 s1 = __floats2bfloat162_rn(__uint_as_float(w[2]), __uint_as_float(w[3]));
                    uint2 sv;
                    sv.x = *reinterpret_cast<const uint32_t *>(&s0);
                    sv.y = *reinterpret_cast<const uint32_t *>(&s1);
                    reinterpret_cast<uint2 *>(Tsh + (c - lo) * (row_bytes / 4))[u] = sv;
                }
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        nmax = fmaxf(nmax, ss);
    }
    // the lane's mu partial -> its columns of the warp's smem row (each column owned by one lane)
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int u = h2 * 64 + q * 32 + lane;
            if (u >= nvec) continue;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if (dtype == 0) {
                    if (h2 == 0) {
                        smu[wib][u * 8 + 2 * i] = acc[q * 8 + 2 * i];
                        smu[wib][u * 8 + 2 * i + 1] = acc[q * 8 + 2 * i + 1];
                    }
                } else {
                    smu[wib][u * 4 + i] = acc[h2 * 8 + q * 4 + i];
                }
            }
        }
    mu_block_flush(smu, (row_bytes / 16) * epv, mu_fx);
    // one atomic per block for the running norm bound (the softmax reference, R1)
    if (lane == 0) wmax[wib] = nmax;
    __syncthreads();
    if (threadIdx.x == 0) {
        float mx = 0.f;
        for (int i = 0; i < (blockDim.x >> 5); ++i) mx = fmaxf(mx, wmax[i]);
        float nrm = sqrtf(mx);
        if (!(nrm <= 3.0e38f)) nrm = 3.0e38f;
        if (nrm > 0.f) atomicMax(&sc->tmax_bits, __float_as_int(nrm));
    }
}

// K >= 2 features per slot (NEXT-1).  The center of a slot is the exact mean
// T_bar_c = (1/K) sum_k T[c,k] (Eq. 8): its fp32 value, computed always in this order (fp32
// sum over k from 0, then one multiply by 1/K; exact for K = 2 and K = 4 with bf16 features),
// gives w_c = 1/||T_bar_c|| (reading R4) and the slot's mu contribution w_c T_bar_c (R3).  The
// logits GEMM contracts x with the K raw rows (1/K folded into a_r), so the logits use the
// exact mean too; only the P x pool GEMM and the combine read the bf16 rounding of T_bar
// (R5).  Lane l holds columns 32 e + l (e < 16) of a d <= 512 row.
__device__ __forceinline__ float slot_mean16(const __nv_bfloat16 *__restrict__ raw, int K, int d, int lane,
                                             float (&mf)[16]) {
    const float invK = 1.0f / static_cast<float>(K);
    float ss = 0.f;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
        const int col = e * 32 + lane;
        float acc = 0.f;
        if (col < d)
            for (int kk = 0; kk < K; ++kk) acc = __fadd_rn(acc, __bfloat162float(raw[kk * d + col]));
        mf[e] = __fmul_rn(acc, invK);
        ss = __fmaf_rn(mf[e], mf[e], ss);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ss = __fadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, o));
    return ss;  // ||T_bar_c||^2 in every lane
}
__device__ __forceinline__ float slot_weight(float ss) { return ss > 0.f ? rsqrtf(ss) : 0.f; }

// One warp per block row: the K raw rows are copied bit-exactly (state / checkpoint), the bf16
// T_bar and w_c written, and mu updated by (new - old) contributions -- the old one recomputed
// from the slot's raw rows before they are overwritten (same arithmetic as when it was added).
__global__ void __launch_bounds__(256) k_enqueue_k(const __nv_bfloat16 *__restrict__ g, const int64_t *__restrict__ y,
                                                   int64_t m_glob, int K, int d, int64_t E, int64_t C,
                                                   int64_t lo, int64_t hi, __nv_bfloat16 *__restrict__ Traw,
                                                   __nv_bfloat16 *__restrict__ Tbar, float *__restrict__ wslot,
                                                   int64_t *__restrict__ lab, Scalars *sc,
                                                   const int64_t *__restrict__ dst_seq,
                                                   unsigned long long *__restrict__ mu_fx, int64_t occ_before,
                                                   LabelIndex ix) {
    __shared__ float wmax[8];
    __shared__ long long smu[MU_WARPS][512];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    enqueue_labels(y, m_glob, E, C, lo, hi, lab, dst_seq, ix);
    mu_block_init(smu, d);
    float nmax = 0.f;
    const int64_t e0 = E % C;
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + wib; j < m_glob; j += nwarps) {
        const int64_t c = enq_slot(j, e0, C, dst_seq);
        if (c < lo || c >= hi) continue;
        const int64_t yl = y[j];
        if (yl < 0) {
            if (lane == 0) latch(sc, ERR_DEVICE, DET_BAD_LABEL);
            continue;
        }
        __nv_bfloat16 *dst = Traw + (c - lo) * K * d;
        float mf[16];
        if (c < occ_before) {  // an occupied slot: its contribution leaves (wold = 0: zero center)
            const float wold = wslot[c - lo];
            slot_mean16(dst, K, d, lane, mf);
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const int col = e * 32 + lane;
                if (col < d) smu[wib][col] -= mu_fx_of(__fmul_rn(wold, mf[e]));
            }
        }
        __syncwarp();  // (every lane has read the old rows)
        {   // 16-byte vector copy (rows of K d bf16 are multiples of 256 B, 16-B aligned)
            const int4 *src = reinterpret_cast<const int4 *>(g + j * K * d);
            int4 *d4 = reinterpret_cast<int4 *>(dst);
            for (int i = lane; i < K * d / 8; i += 32) d4[i] = __ldcs(src + i);
        }
        __syncwarp();
        const float ss = slot_mean16(dst, K, d, lane, mf);
        const float wv = slot_weight(ss);
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int col = e * 32 + lane;
            if (col < d) {
                Tbar[(c - lo) * d + col] = __float2bfloat16_rn(mf[e]);
                smu[wib][col] += mu_fx_of(__fmul_rn(wv, mf[e]));
            }
        }
        if (lane == 0) wslot[c - lo] = wv;
        nmax = fmaxf(nmax, ss);
    }
    mu_block_flush(smu, d, mu_fx);
    if (lane == 0) wmax[wib] = nmax;
    __syncthreads();
    if (threadIdx.x == 0) {
        float mx = 0.f;
        for (int i = 0; i < (blockDim.x >> 5); ++i) mx = fmaxf(mx, wmax[i]);
        float nrm = sqrtf(mx);
        if (!(nrm <= 3.0e38f)) nrm = 3.0e38f;
        if (nrm > 0.f) atomicMax(&sc->tmax_bits, __float_as_int(nrm));
    }
}

// set_state with K >= 2: rebuild T_bar, w and the norm bound from the raw features (one warp
// per slot, the same arithmetic as k_enqueue_k)
__global__ void __launch_bounds__(256) k_rebuild_k(const __nv_bfloat16 *__restrict__ Traw, int64_t rows, int K, int d,
                                                   __nv_bfloat16 *__restrict__ Tbar, float *__restrict__ wslot,
                                                   Scalars *sc) {
    const int lane = threadIdx.x & 31;
    const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (r >= rows) return;
    float mf[16];
    const float ss = slot_mean16(Traw + r * K * d, K, d, lane, mf);
#pragma unroll
    for (int e = 0; e < 16; ++e) {
        const int col = e * 32 + lane;
        if (col < d) Tbar[r * d + col] = __float2bfloat16_rn(mf[e]);
    }
    if (lane == 0) {
        wslot[r] = slot_weight(ss);
        const float nrm = sqrtf(ss);
        if (nrm > 0.f) atomicMax(&sc->tmax_bits, __float_as_int(nrm));
    }
}

// set_state with K >= 2: mu over the restored slots [0, rows) of the shard from scratch (one
// warp per slot, the same per-slot contributions as k_enqueue_k)
__global__ void __launch_bounds__(256) k_mu_sum_k(const __nv_bfloat16 *__restrict__ Traw, const float *__restrict__ wslot,
                                                  int64_t rows, int K, int d, unsigned long long *__restrict__ mu_fx) {
    __shared__ long long smu[MU_WARPS][512];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    mu_block_init(smu, d);
    for (int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + wib; r < rows;
         r += static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5)) {
        float mf[16];
        slot_mean16(Traw + r * K * d, K, d, lane, mf);
        const float w = wslot[r];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int col = e * 32 + lane;
            if (col < d) smu[wib][col] += mu_fx_of(__fmul_rn(w, mf[e]));
        }
    }
    mu_block_flush(smu, d, mu_fx);
}

// ------------------------------------------------------------------ the pool sum mu (L_cos)
// set_state: mu over the restored slots from scratch (the same per-slot contributions as the
// enqueue kernels' running sum).  Rows m of the call -> slot (dst_seq ? dst_seq[m] : E + m)
// mod C, skipped outside [lo, hi); sign -1 subtracts.  Thread t owns columns 2t, 2t+1; each
// CTA adds its column sums with one atomic each.
__global__ void __launch_bounds__(256) k_mu_sum(const uint8_t *__restrict__ T, int dtype, const float *__restrict__ wslot,
                                                int d, int64_t m, int64_t E, int64_t C, int64_t lo, int64_t hi,
                                                const int64_t *__restrict__ dst_seq, int sign,
                                                unsigned long long *__restrict__ mu_fx) {
    const int c0 = 2 * threadIdx.x;
    long long acc0 = 0, acc1 = 0;
    for (int64_t j = blockIdx.x; j < m; j += gridDim.x) {
        const int64_t c = (dst_seq ? dst_seq[j] : E + j) % C;
        if (c < lo || c >= hi || c0 >= d) continue;
        const int64_t sl = c - lo;
        float v0, v1;
        if (dtype == 0) {  // bf16 (T_bar for K >= 2)
            const uint32_t u = *reinterpret_cast<const uint32_t *>(T + (sl * d + c0) * 2);
            v0 = __uint_as_float(u << 16);
            v1 = __uint_as_float(u & 0xffff0000u);
        } else {
            const float2 f = *reinterpret_cast<const float2 *>(T + (sl * d + c0) * 4);
            v0 = f.x;
            v1 = f.y;
        }
        if (wslot) {
            const float w = wslot[sl];
            v0 = __fmul_rn(w, v0);
            v1 = __fmul_rn(w, v1);
        }
        acc0 += mu_fx_of(v0);
        acc1 += mu_fx_of(v1);
    }
    if (c0 < d && (acc0 | acc1)) {
        atomicAdd(mu_fx + c0, static_cast<unsigned long long>(sign * acc0));
        atomicAdd(mu_fx + c0 + 1, static_cast<unsigned long long>(sign * acc1));
    }
}

// recompute the norm bound over a whole shard (after set_state)
__global__ void k_pool_norm_max(const uint8_t *__restrict__ T, int64_t rows, int row_bytes,
                                int dtype, Scalars *sc) {
    const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const int4 *src = reinterpret_cast<const int4 *>(T + r * row_bytes);
    float ss = 0.f;
    for (int u = lane; u < row_bytes / 16; u += 32) {
        int4 v = src[u];
        const uint32_t w[4] = {static_cast<uint32_t>(v.x), static_cast<uint32_t>(v.y),
                               static_cast<uint32_t>(v.z), static_cast<uint32_t>(v.w)};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (dtype == 0) {
                float a = __uint_as_float(w[i] << 16), b = __uint_as_float(w[i] & 0xffff0000u);
                ss += a * a + b * b;
            } else {
                float a = __uint_as_float(w[i]);
                ss += a * a;
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) {
        float nrm = sqrtf(ss);
        if (!(nrm <= 3.0e38f)) nrm = 3.0e38f;
        atomicMax(&sc->tmax_bits, __float_as_int(nrm));
    }
}

// ------------------------------------------------------------------ a10: G-Net EMA
// g <- m*g + (1-m)*p in fp64 (__dmul_rn/__dadd_rn: no contraction), RNE to fp32.
__device__ __forceinline__ float ema1(float gv, float pv, double m, double om) {
    return __double2float_rn(__dadd_rn(__dmul_rn(m, static_cast<double>(gv)),
                                       __dmul_rn(om, static_cast<double>(pv))));
}
// One CTA per 256 float4 (4 KB of g): short-lived CTAs, so a concurrently launched
// persistent kernel (the fused loss kernel) gets its SMs back within microseconds when the
// EMA runs on a side stream; four independent 16-B loads per thread in flight (two of p, two
// of g).  (Measured: 4 float4 per array per thread, or 160 / 192-thread CTAs, were slower.)
// Small CTAs (128 threads, <= 40 registers, no smem) fit next to the fused loss kernel on an
// SM (its CTA leaves ~6K registers and ~24 KB of smem free), so an EMA on a side stream can run
// concurrently with it instead of waiting for its SMs.
constexpr int EMA_PER_THREAD = 2;
constexpr int EMA_THREADS = 128;
__global__ void __launch_bounds__(EMA_THREADS, 12) k_ema(const float4 *__restrict__ p, float4 *__restrict__ g, int64_t n4,
                                                        double m, double om) {
    const int64_t base = static_cast<int64_t>(blockIdx.x) * (EMA_THREADS * EMA_PER_THREAD) + threadIdx.x;
    float4 a[EMA_PER_THREAD], b[EMA_PER_THREAD];
#pragma unroll
    for (int u = 0; u < EMA_PER_THREAD; ++u) {
        const int64_t i = base + u * EMA_THREADS;
        if (i < n4) {
            a[u] = __ldcs(p + i);
            b[u] = __ldcs(g + i);
        }
    }
#pragma unroll
    for (int u = 0; u < EMA_PER_THREAD; ++u) {
        const int64_t i = base + u * EMA_THREADS;
        if (i < n4) {
            float4 v = b[u];
            v.x = ema1(v.x, a[u].x, m, om);
            v.y = ema1(v.y, a[u].y, m, om);
            v.z = ema1(v.z, a[u].z, m, om);
            v.w = ema1(v.w, a[u].w, m, om);
            __stcs(g + i, v);
        }
    }
}
__global__ void k_ema_tail(const float *__restrict__ p, float *__restrict__ g, int64_t lo, int64_t n,
                           double m, double om) {
    const int64_t i = lo + threadIdx.x;
    if (i < n) g[i] = ema1(g[i], p[i], m, om);
}

// ------------------------------------------------------------------ a3: target resolve
// Hash table of the batch labels (open addressing, H a power of two >= 2N).
__global__ void k_hash_clear(int64_t *keys, unsigned long long *vals, int H) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < H; i += gridDim.x * blockDim.x) {
        keys[i] = -1;
        vals[i] = 0ull;
    }
}

// a2 + a3 (part 1): per row (one warp): 1/||x_i|| and insert y_i into the hash table.
template <typename T>
__global__ void k_rownorm_insert(const T *__restrict__ x, const int64_t *__restrict__ y, int64_t N,
                                 int d, float *__restrict__ inv_n, int64_t *keys, int H,
                                 int *__restrict__ hslot, Scalars *sc, LabelIndex ix,
                                 int64_t *__restrict__ tseq) {
    const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= N) return;
    // the two label lookups first, on their own lanes (their dependent round trips overlap each
    // other and the row's loads): lane 1 -- the shard's label index (a3: the target = the label's
    // newest slot of this shard, D8); lane 2 -- the batch-label hash (stale-duplicate lists, R8)
    const int64_t key = y[i];
    if (key < 0) {
        if (lane == 0) {
            latch(sc, ERR_DEVICE, DET_BAD_LABEL);
            hslot[i] = -1;
            tseq[i] = -1;
        }
    } else if (lane == 1) {
        tseq[i] = idx_lookup(ix, key);
    } else if (lane == 2) {
        unsigned h = static_cast<unsigned>(hash64(static_cast<uint64_t>(key))) & (H - 1);
        for (;;) {
            unsigned long long old = atomicCAS(reinterpret_cast<unsigned long long *>(keys + h),
                                               static_cast<unsigned long long>(-1ll),
                                               static_cast<unsigned long long>(key));
            if (old == static_cast<unsigned long long>(-1ll) ||
                old == static_cast<unsigned long long>(key))
                break;
            h = (h + 1) & (H - 1);
        }
        hslot[i] = static_cast<int>(h);
    }
    float ss = 0.f;
    {  // 16-byte vector loads (d is a multiple of 128, rows 16-byte aligned)
        const uint4 *row = reinterpret_cast<const uint4 *>(x + i * d);
        const int nvec = d * static_cast<int>(sizeof(T)) / 16;
        for (int u = lane; u < nvec; u += 32) {
            const uint4 v = row[u];
            const uint32_t q[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (sizeof(T) == 2) {
                    const float lo = __uint_as_float(q[e] << 16), hi = __uint_as_float(q[e] & 0xffff0000u);
                    ss += lo * lo + hi * hi;
                } else {
                    const float f = __uint_as_float(q[e]);
                    ss += f * f;
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) {
        float nrm = sqrtf(ss);
        if (!(nrm > 0.f) || !(nrm <= 3.0e38f)) {
            latch(sc, ERR_DEVICE, DET_ZERO_ROW);
            inv_n[i] = 0.f;
        } else {
            inv_n[i] = 1.0f / nrm;
        }
    }
}

// ------------------------------------------------------------------ NEXT-3: refresh-in-place enqueue
// SPEC's insert_batch (reading R7): a block row whose label is resident
// overwrites that slot's features in place (age kept); the other rows are appended at
// E, E+1, ... in block order -- together with the resident rows whose slot those appends
// would overwrite (the smallest fixed point n = n0 + #{sigma_j < E + n - C}).  The block's
// labels go into their own hash (k_blk_insert: the S:277 duplicate check), sigma_j = newest write
// index (-1 = not resident) comes from the shard's label index (k_idx_lookup; W > 1: MAX
// all-reduce), and one CTA plans the destinations (k_refresh_plan).
__global__ void k_blk_insert(const int64_t *__restrict__ y, int64_t M, int64_t *keys, int H,
                             int *__restrict__ hslot, Scalars *sc) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= M) return;
    const int64_t key = y[j];
    if (key < 0) {
        latch(sc, ERR_DEVICE, DET_BAD_LABEL);
        hslot[j] = -1;
        return;
    }
    unsigned h = static_cast<unsigned>(hash64(static_cast<uint64_t>(key))) & (H - 1);
    for (;;) {
        const unsigned long long old = atomicCAS(reinterpret_cast<unsigned long long *>(keys + h),
                                                 static_cast<unsigned long long>(-1ll),
                                                 static_cast<unsigned long long>(key));
        if (old == static_cast<unsigned long long>(-1ll)) break;
        if (old == static_cast<unsigned long long>(key)) {  // ids pairwise distinct
            latch(sc, ERR_DEVICE, DET_DUP_BLOCK);
            break;
        }
        h = (h + 1) & (H - 1);
    }
    hslot[j] = static_cast<int>(h);
}

// single CTA: the fixed point n, then dst_seq[j] (write index of row j's slot) and
// sc->n_app = n; clears the block hash for the next call
__global__ void __launch_bounds__(1024) k_refresh_plan(const int64_t *__restrict__ sigma, int64_t M, int64_t E,
                                                       int64_t C, int64_t *__restrict__ dst_seq, Scalars *sc,
                                                       int64_t *keys, unsigned long long *vals, int H) {
    __shared__ int wsum[32];
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, w = tid >> 5;
    const int64_t per = (M + nt - 1) / nt;
    const int64_t r0 = tid * per, r1 = r0 + per < M ? r0 + per : M;
    auto block_sum = [&](int v) {  // all threads get the total
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        __syncthreads();
        if (lane == 0) wsum[w] = v;
        __syncthreads();
        int t = 0;
        for (int i = 0; i < (nt >> 5); ++i) t += wsum[i];
        return t;
    };
    int c0 = 0;
    for (int64_t j = r0; j < r1; ++j) c0 += sigma[j] < 0;
    const int n0 = block_sum(c0);
    long long n = n0;
    for (;;) {
        int c = 0;
        for (int64_t j = r0; j < r1; ++j) c += sigma[j] >= 0 && sigma[j] < E + n - C;
        const long long f = n0 + block_sum(c);
        if (f == n) break;
        n = f;
    }
    // exclusive scan of the appended flags in block order
    int cnt = 0;
    for (int64_t j = r0; j < r1; ++j) cnt += sigma[j] < 0 || sigma[j] < E + n - C;
    int v = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    __syncthreads();
    if (lane == 31) wsum[w] = v;
    __syncthreads();
    if (w == 0) {
        int s2 = lane < (nt >> 5) ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, s2, o);
            if (lane >= o) s2 += t;
        }
        wsum[lane] = s2;
    }
    __syncthreads();
    long long k = (w > 0 ? wsum[w - 1] : 0) + v - cnt;
    for (int64_t j = r0; j < r1; ++j) {
        const int64_t sg = sigma[j];
        dst_seq[j] = (sg < 0 || sg < E + n - C) ? E + k++ : sg;
    }
    if (tid == 0) sc->n_app = n;
    for (int h = tid; h < H; h += nt) {
        keys[h] = -1;
        vals[h] = 0ull;
    }
}

// ------------------------------------------------------------------ NEXT-3: stale self-duplicates
// Variant "exclude stale self-duplicates" (D8 keeps them): an in-pool
// row's softmax skips the occupied slots that carry its own label but are not its target
// (the newest such slot).  Built after the targets are final (W > 1: after C2): a per-tile
// list of the shard's stale slots, (local slot, label hash entry), in tile order, which the
// fused kernel's softmax warps consult once per tile.  Two passes over the shard's labels
// (count per 128-slot tile, then fill) around an exclusive scan of the tile counts.
__device__ __forceinline__ int stale_dup_entry(int64_t L, int64_t c, int64_t C, int64_t E,
                                               const int64_t *__restrict__ keys, int H,
                                               const int64_t *__restrict__ hgseq) {
    if (L < 0) return -1;
    unsigned h = static_cast<unsigned>(hash64(static_cast<uint64_t>(L))) & (H - 1);
    for (;;) {
        const int64_t k = keys[h];
        if (k == -1) return -1;
        if (k == L) {
            const int64_t seq = c + C * ((E - 1 - c) / C);
            return seq != hgseq[h] ? static_cast<int>(h) : -1;
        }
        h = (h + 1) & (H - 1);
    }
}

__global__ void k_dup_count(const int64_t *__restrict__ lab, int64_t n_occ_loc, int64_t lo, int64_t C,
                            int64_t E, const int64_t *__restrict__ keys, int H,
                            const int64_t *__restrict__ hgseq, int *__restrict__ tile_cnt) {
    for (int64_t cl = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; cl < n_occ_loc;
         cl += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (stale_dup_entry(lab[cl], lo + cl, C, E, keys, H, hgseq) >= 0) atomicAdd(tile_cnt + (cl >> 7), 1);
}

// single CTA: tile_off[t] = sum of tile_cnt[< t] (n_tiles + 1 entries); tile_cnt reset to 0
// for use as the fill cursor
__global__ void __launch_bounds__(1024) k_dup_scan(int *__restrict__ tile_cnt, int *__restrict__ tile_off,
                                                   int n_tiles) {
    __shared__ int wsum[32];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int per = (n_tiles + nt - 1) / nt;
    const int t0 = tid * per, t1 = min(t0 + per, n_tiles);
    int cnt = 0;
    for (int t = t0; t < t1; ++t) cnt += tile_cnt[t];
    const int lane = tid & 31, w = tid >> 5;
    int v = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    if (lane == 31) wsum[w] = v;
    __syncthreads();
    if (w == 0) {
        int s2 = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int u = __shfl_up_sync(0xffffffffu, s2, o);
            if (lane >= o) s2 += u;
        }
        wsum[lane] = s2;
    }
    __syncthreads();
    int run = (w > 0 ? wsum[w - 1] : 0) + v - cnt;
    for (int t = t0; t < t1; ++t) {
        tile_off[t] = run;
        run += tile_cnt[t];
        tile_cnt[t] = 0;
    }
    if (tid == nt - 1) tile_off[n_tiles] = wsum[31];
}

__global__ void k_dup_fill(const int64_t *__restrict__ lab, int64_t n_occ_loc, int64_t lo, int64_t C,
                           int64_t E, const int64_t *__restrict__ keys, int H,
                           const int64_t *__restrict__ hgseq, int *__restrict__ tile_cur,
                           const int *__restrict__ tile_off, int2 *__restrict__ list) {
    for (int64_t cl = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; cl < n_occ_loc;
         cl += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int he = stale_dup_entry(lab[cl], lo + cl, C, E, keys, H, hgseq);
        if (he >= 0) {
            const int t = static_cast<int>(cl >> 7);
            list[tile_off[t] + atomicAdd(tile_cur + t, 1)] = make_int2(static_cast<int>(cl), he);
        }
    }
}

// ------------------------------------------------------------------ a3: split + compaction
// Single CTA (1024 threads): Eq. 6's split into in-pool (F_p^DCP) and out-of-pool
// rows, compaction of the in-pool rows in batch order, per-row softmax coefficients,
// the pairing check (D13), and coefficients (0, +inf) -- p = 0 -- for the padding rows.
struct CompactArgs {
    const int64_t *tseq;      // [N] global write index of the target or -1 (the label index lookup;
                              // W > 1: after the MAX all-reduce)
    const float *inv_n;       // [N]
    const int32_t *pairing;   // [N] or null
    int64_t N, C, lo, hi, E, M_last;
    float s, log2e_s;         // s, s*log2(e)
    float a_scale;            // 1/K: GEMM 1 sums the K raw rows of a slot (NEXT-1), a_r takes the 1/K
    int R_max;
    int neg_mode;             // 0: mu path; 1 (hinge) / 2 (max): out-of-pool rows are compacted
                              // after the in-pool rows (index neg0 + j, neg0 = n_pos rounded up to 32) and run through the kernel
    int *comp_idx;            // [N]: k >= 0 in-pool row k; -1 out-of-pool (mu path); -2 - k
                              // out-of-pool row compacted at k (neg_mode != 0)
    int *pos_row;             // [R_max]
    float2 *row_ab;           // [R_max]
    int *row_tgt;             // [R_max]
    float *ttgt;              // [R_max]
    Scalars *sc;
    const int *tmax_bits;     // max ||T_c|| over the whole pool (all shards)
    float ref_scale;          // s*log2(e)*(1+2^-10): reference exponent per unit norm
    // NEXT-3 "exclude stale self-duplicates": the row's label hash entry (-1 = none) and the
    // target write index per hash entry, read by the duplicate-list kernels below
    const int64_t *blk_seq;   // [M_last] after a refresh-in-place enqueue, else null
    int excl;
    const int *hslot;         // [N]
    int *row_hent;            // [R_max]
    int64_t *hgseq;           // [H]
    int G_pc, n_tiles_pc;     // dcp_pc_kernel's clusters and tiles: choose its S here (G_pc = 0: other kernels)
    int rg_pc;                // rows per group of that kernel: 128 (dcp_pc_kernel) or 256 (dcp_pc4_kernel)
    int seg_cap;              // segments of rg_pc rows the partial buffers hold (dcp_pc4_kernel)
};
__global__ void __launch_bounds__(1024) k_compact(CompactArgs a) {
    // CTA b compacts rows [b*1024, (b+1)*1024).  Every CTA counts the in-pool rows of the
    // whole batch (n_pos) and of the rows before its chunk (its base) in one coalesced pass
    // (N int64 from L2), so the chunks are independent.
    __shared__ int wsum[32], wpre_s[32];
    __shared__ int s_tot, s_before;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, w = tid >> 5;
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * nt;
    auto tseq_of = [&](int64_t i) -> int64_t { return a.tseq[i]; };
    int cnt = 0, before = 0;
    for (int64_t i = tid; i < a.N; i += nt) {
        const int f = tseq_of(i) >= 0;
        cnt += f;
        before += (i < c0) ? f : 0;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        before += __shfl_xor_sync(0xffffffffu, before, o);
    }
    if (lane == 0) {
        wsum[w] = cnt;
        wpre_s[w] = before;
    }
    __syncthreads();
    if (tid == 0) {
        int t = 0, b = 0;
        for (int q = 0; q < (nt >> 5); ++q) {
            t += wsum[q];
            b += wpre_s[q];
        }
        s_tot = t;
        s_before = b;
    }
    __syncthreads();
    const int n_pos = s_tot;
    const int neg0 = a.neg_mode ? (n_pos + 31) & ~31 : n_pos;
    const float tmax = __int_as_float(*a.tmax_bits);
    const float B = a.ref_scale * tmax;
    // this CTA's chunk, one row per thread; k = in-pool rows before row i (ballot scan)
    {
        const int64_t i = c0 + tid;
        const int64_t ts = i < a.N ? tseq_of(i) : -1;
        const bool f = i < a.N && ts >= 0;
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        __syncthreads();  // (wsum reuse)
        if (lane == 0) wsum[w] = __popc(bal);
        __syncthreads();
        int wpre = 0;
        for (int q = 0; q < w; ++q) wpre += wsum[q];
        const int k = s_before + wpre + __popc(bal & ((1u << lane) - 1u));
        if (i < a.N) {
            if (a.pairing && a.pairing[i] >= 0) {
                const bool inb = a.pairing[i] < a.M_last;
                // pure Eq. 7: block row j sits at write index E - M_last + j; after a
                // refresh-in-place enqueue (NEXT-3) at the planned blk_seq[j]
                const int64_t want = !inb ? -2 : (a.blk_seq ? a.blk_seq[a.pairing[i]] : a.E - a.M_last + a.pairing[i]);
                if (!inb || ts != want) latch(a.sc, ERR_PAIRING, DET_PAIRING);
            }
            if (ts < 0 && a.neg_mode) {
                const int kn = neg0 + static_cast<int>(i - k);  // i - k = out-of-pool rows before i
                a.comp_idx[i] = -2 - kn;
                a.pos_row[kn] = static_cast<int>(i);
                a.row_ab[kn] = make_float2(a.inv_n[i] * a.a_scale, 0.f);  // e = <x, T_bar> / ||x|| = cosine
                a.row_tgt[kn] = -2;
                a.ttgt[kn] = -INFINITY;
            } else if (ts >= 0) {
                a.comp_idx[i] = k;
                a.pos_row[k] = static_cast<int>(i);
                if (a.excl) {
                    const int he = a.hslot[i];
                    a.row_hent[k] = he;
                    if (he >= 0) a.hgseq[he] = ts;  // rows sharing a label share the target
                }
                a.row_ab[k] = make_float2(a.log2e_s * a.inv_n[i] * a.a_scale, B);
                const int64_t slot = ts % a.C;
                a.row_tgt[k] = (slot >= a.lo && slot < a.hi) ? static_cast<int>(slot - a.lo) : -1;
                a.ttgt[k] = -INFINITY;
            } else {
                a.comp_idx[i] = -1;
            }
        }
    }
    if (blockIdx.x != 0) return;
    // (CTA 0) the padding rows of the last row group (the mu vector of the L_cos gradient is
    // not a kernel row: it is kept incrementally by the enqueue, k_mu_sum)
    const int n_rows = a.neg_mode ? neg0 + static_cast<int>(a.N) - n_pos : n_pos;
    if (a.excl)
        for (int r = n_pos + tid; r < a.R_max; r += nt) a.row_hent[r] = -1;  // out-of-pool, padding
    // padding rows (up to neg0, and after n_rows): e = -inf, so p = 0 (zero P operand in GEMM 2)
    for (int r = n_pos + tid; r < a.R_max; r += nt) {
        if (r >= neg0 && r < n_rows) continue;  // (out-of-pool rows, written above)
        a.row_ab[r] = make_float2(0.f, INFINITY);
        a.row_tgt[r] = -1;
        a.ttgt[r] = -INFINITY;
    }
    if (a.G_pc > 0) {  // dcp_pc_kernel's S: one candidate per thread, argmin (cost, then S)
        __shared__ unsigned long long best;
        if (tid == 0) best = ~0ull;
        __syncthreads();
        const int R = (n_rows + a.rg_pc - 1) / a.rg_pc;
        int s_hi = pc_s_hi(R, a.G_pc, a.n_tiles_pc);
        if (a.rg_pc != PC_R && R > 0 && s_hi > a.seg_cap / R) s_hi = a.seg_cap / R < 1 ? 1 : a.seg_cap / R;
        for (int S = tid + 1; S <= s_hi; S += nt) {
            const float c = pc_sched_cost(S, R, a.G_pc, a.n_tiles_pc);
            atomicMin(&best, (static_cast<unsigned long long>(__float_as_uint(c)) << 32) | static_cast<unsigned>(S));
        }
        __syncthreads();
        if (tid == 0) {
            int S = static_cast<int>(best & 0xffffffffull);
            if (g_force_S > 0) S = g_force_S < s_hi ? g_force_S : s_hi;  // (timing experiments; within the layout's bounds)
            if (S > a.n_tiles_pc) S = a.n_tiles_pc;
            a.sc->S_sched = S < 1 ? 1 : S;
        }
    }
    if (tid == 0) {
        a.sc->refine = 0;
        a.sc->neg0 = neg0;
        a.sc->n_rows = n_rows;
        a.sc->n_pos = n_pos;
        a.sc->n_neg = static_cast<int>(a.N) - n_pos;
        a.sc->n_pos_sum += static_cast<unsigned long long>(n_pos);
    }
}

// Gather the in-pool rows into the dense bf16 operand X_pos, and set the row's softmax
// reference (R1): b_r = max(z_t, bound - 100) in log2 units, where z_t = a_r <x_r, T_t>
// is the unmargined target logit (computed by the shard that owns the target slot; other
// shards keep bound - 100).  Every exponent is then <= 100 (no overflow of p or O), and
// the dominant terms stay representable for any |cos| <= 1 at s <= 76.
__global__ void __launch_bounds__(256) k_gather(const uint8_t *__restrict__ x, const int *__restrict__ pos_row,
                                                const Scalars *__restrict__ sc, int row_bytes,
                                                uint8_t *__restrict__ Xp, const uint8_t *__restrict__ T,
                                                const int *__restrict__ row_tgt, float2 *__restrict__ row_ab,
                                                float kf, int f32) {
    // one warp per compacted row, 8 rows per CTA
    const int k = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (k >= sc->n_rows || (k >= sc->n_pos && k < sc->neg0)) {
        // the padding rows of the last row group: zero operands (their
        // products are discarded; zeros keep the tensor pipe's switching power down)
        if (k < ((sc->n_rows + 255) & ~255)) {  // (256-row groups of dcp_pc4_kernel)
            int4 *dst = reinterpret_cast<int4 *>(Xp + static_cast<int64_t>(k) * row_bytes);
            for (int u = lane; u < row_bytes / 16; u += 32) dst[u] = make_int4(0, 0, 0, 0);
        }
        return;
    }
    const int4 *src = reinterpret_cast<const int4 *>(x + static_cast<int64_t>(pos_row[k]) * row_bytes);
    int4 *dst = reinterpret_cast<int4 *>(Xp + static_cast<int64_t>(k) * row_bytes);
    const int ts = row_tgt[k];  // local target slot, -1 (not on this shard), -2 (out-of-pool row)
    const int4 *tr = reinterpret_cast<const int4 *>(T + static_cast<int64_t>(ts < 0 ? 0 : ts) * row_bytes);
    float dot = 0.f;
    for (int u = lane; u < row_bytes / 16; u += 32) {
        const int4 v = src[u];
        dst[u] = v;
        if (ts >= 0) {
            const int4 w = tr[u];
            const uint32_t a[4] = {static_cast<uint32_t>(v.x), static_cast<uint32_t>(v.y),
                                   static_cast<uint32_t>(v.z), static_cast<uint32_t>(v.w)};
            const uint32_t b[4] = {static_cast<uint32_t>(w.x), static_cast<uint32_t>(w.y),
                                   static_cast<uint32_t>(w.z), static_cast<uint32_t>(w.w)};
            if (f32) {
#pragma unroll
                for (int i = 0; i < 4; ++i) dot += __uint_as_float(a[i]) * __uint_as_float(b[i]);
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    dot += __uint_as_float(a[i] << 16) * __uint_as_float(b[i] << 16) +
                           __uint_as_float(a[i] & 0xffff0000u) * __uint_as_float(b[i] & 0xffff0000u);
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (lane == 0 && ts != -2) {  // (-2: out-of-pool row of NEXT-3, (a, b) final)
        float2 ab = row_ab[k];
        const float floor_b = ab.y - 100.f;  // ab.y holds the global bound on entry
        const float zt = ab.x * dot * kf;  // (a_r carries 1/K, T holds the mean: K = 1 for one feature)
        ab.y = ts >= 0 ? fmaxf(zt, floor_b) : floor_b;
        row_ab[k] = ab;
    }
}

// ------------------------------------------------------------------ a6 + a8 + a9: combine
// One CTA per global row.  Sums the main kernel's segment partials in a fixed order,
// forms dL/dx_hat (Eq. 9 gradient with the target term in fp64, D12), or the L_cos
// gradient mu / (N_neg C_occ) for out-of-pool rows (D10), applies the normalisation
// Jacobian and writes dx in the input dtype, plus the per-row loss terms.
struct CombineArgs {
    const uint8_t *x;           // [N, d] dtype
    const float *inv_n;         // [N]
    const int *comp_idx;        // [N]
    const float2 *row_ab;       // [R_max]
    const int *row_tgt;         // [R_max] (local slot)
    const float *ttgt;          // [R_max]
    const float *seg_l, *seg_mx, *seg_O;
    const uint8_t *T;           // local pool, bf16 (an fp32 pool's bf16 shadow: the operand of GEMM 2)
    // the exact center of a slot for the gradient's target / hardest-negative rows: the bf16 row (K = 1),
    // the fp32 row of an fp32 pool (D21), or the fp32 mean of the K raw rows (R5)
    const uint8_t *Tc;
    int Tc_kind;                // 0 bf16 rows (= T), 1 fp32 rows, 2 K raw bf16 rows per slot
    int Kc;
    const Scalars *sc;
    Scalars *sc_w;
    int64_t N, C_occ;
    int d, dtype, G, n_tiles;
    int rows_per_group;         // 64 (TP64 kernel) or 128 (producer/consumer kernel)
    int wide;                   // the partials come from dcp_pc_kernel / dcp_pc4_kernel: their S is sc->S_sched
    float s, margin_l2;
    uint8_t *dx;                // [N, d] dtype
    double *rowloss;            // [N]
    float *st_lse, *st_cos, *st_phi, *st_ell;  // [N] row statistics
    // NEXT-3 L_cos variants: reduction (mean: 1/C_occ, sum: 1), hinge, weight lambda;
    // neg_mode 1 (hinge) / 2 (max) reads the out-of-pool rows' own kernel partials
    int neg_mode, phi_mean, hinge, my_rank;
    float lam;
    const int *seg_arg;         // [S][128] local argmax slot of a segment (neg_mode 2)
    const float *wslot;         // [C_loc] 1/||T_bar_c|| (K >= 2) or null
    const long long *mu_fx;     // [d] this shard's sum_c w_c T_bar_c, fixed point (k_mu_sum)
    // the batch-label hash, cleared for the next loss call by the final per-row kernel
    // (k_combine / k_finalize_multi: block i clears its slice)
    int64_t *hkeys;
    unsigned long long *hvals;
    int H;
};

// this shard's mu (fixed point -> fp32), the lane's 16 columns in the load_bf16_row layout
__device__ __forceinline__ void load_mu(const CombineArgs &a, int lane, float (&mu)[16]) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int dd = 128 * j + 4 * lane + u;
            mu[4 * j + u] = dd < a.d ? static_cast<float>(static_cast<double>(__ldg(a.mu_fx + dd)) * MU_FX_INV) : 0.f;
        }
}

__device__ __forceinline__ void clear_hash_slice(const CombineArgs &a, int64_t nblk) {
    const int64_t per = (a.H + nblk - 1) / nblk;
    const int64_t h0 = static_cast<int64_t>(blockIdx.x) * per;
    for (int64_t h = h0 + threadIdx.x; h < h0 + per && h < a.H; h += blockDim.x) {
        a.hkeys[h] = -1;
        a.hvals[h] = 0ull;
    }
}

// The per-row kernels below run one WARP per global row (8 rows per 256-thread CTA, no
// block-level synchronisation).  Lane l holds the 16 elements dd = 128 j + 4 l + e
// (j < d/128 <= 4, e < 4) of every d-vector: float4 / 4 x bf16 vector accesses, coalesced.
constexpr int CB_ROWS = 8;  // rows (warps) per CTA
struct RowVec {
    float v[16];
};
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ void zero16(float (&v)[16]) {
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = 0.f;
}
// bf16 row -> fp32 lane elements (times scale)
__device__ __forceinline__ void load_bf16_row(const __nv_bfloat16 *row, int d, int lane, float scale,
                                              float (&v)[16]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int dd = 128 * j + 4 * lane;
        if (dd < d) {
            const uint2 u = *reinterpret_cast<const uint2 *>(row + dd);
            v[4 * j + 0] = __uint_as_float(u.x << 16) * scale;
            v[4 * j + 1] = __uint_as_float(u.x & 0xffff0000u) * scale;
            v[4 * j + 2] = __uint_as_float(u.y << 16) * scale;
            v[4 * j + 3] = __uint_as_float(u.y & 0xffff0000u) * scale;
        } else {
            v[4 * j] = v[4 * j + 1] = v[4 * j + 2] = v[4 * j + 3] = 0.f;
        }
    }
}

// row i of x (dtype: 0 bf16, 1 fp32) -> fp32 lane elements (times scale)
__device__ __forceinline__ void load_x_row(const uint8_t *x, int dtype, int64_t i, int d, int lane, float scale,
                                           float (&v)[16]) {
    if (dtype == 0) {
        load_bf16_row(reinterpret_cast<const __nv_bfloat16 *>(x) + i * d, d, lane, scale, v);
        return;
    }
    const float *row = reinterpret_cast<const float *>(x) + i * d;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int dd = 128 * j + 4 * lane;
        if (dd < d) {
            const float4 u = *reinterpret_cast<const float4 *>(row + dd);
            v[4 * j + 0] = u.x * scale;
            v[4 * j + 1] = u.y * scale;
            v[4 * j + 2] = u.z * scale;
            v[4 * j + 3] = u.w * scale;
        } else {
            v[4 * j] = v[4 * j + 1] = v[4 * j + 2] = v[4 * j + 3] = 0.f;
        }
    }
}
// lane elements -> row i of dx in the input dtype
__device__ __forceinline__ void store_dx_row(uint8_t *dx, int dtype, int64_t i, int d, int lane, const float (&out)[16]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int dd = 128 * j + 4 * lane;
        if (dd >= d) continue;
        if (dtype == 0) {
            const __nv_bfloat162 p0 = __floats2bfloat162_rn(out[4 * j], out[4 * j + 1]);
            const __nv_bfloat162 p1 = __floats2bfloat162_rn(out[4 * j + 2], out[4 * j + 3]);
            uint2 u;
            u.x = *reinterpret_cast<const uint32_t *>(&p0);
            u.y = *reinterpret_cast<const uint32_t *>(&p1);
            *reinterpret_cast<uint2 *>(reinterpret_cast<__nv_bfloat16 *>(dx) + i * d + dd) = u;
        } else {
            *reinterpret_cast<float4 *>(reinterpret_cast<float *>(dx) + i * d + dd) =
                make_float4(out[4 * j], out[4 * j + 1], out[4 * j + 2], out[4 * j + 3]);
        }
    }
}

// sum the partials of compacted row k over its segments (fixed range order);
// the schedule (tp_choose_S) is the main kernel's.  Segments are read in batches of B so
// that the L2 latency is paid once per batch; the accumulation order is the segment order.
__device__ __forceinline__ void gather_row_partials(const CombineArgs &a, int n_rg, int k, float (&o)[16],
                                                    float &lsum, float &mx) {
    const int RG = a.rows_per_group;
    const int rg = k / RG, r = k % RG;
    const int lane = threadIdx.x & 31;
    lsum = 0.f;
    mx = -INFINITY;
    zero16(o);
    if (a.n_tiles <= 0) return;
    const int S = (a.wide ? a.sc->S_sched : tp_choose_S(n_rg, a.G, a.n_tiles));
    constexpr int B = 4;
    for (int s0 = 0; s0 < S; s0 += B) {
        float lv[B], mv[B];
        float4 ov[B][4];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int s = s0 + u;
            lv[u] = 0.f;
            mv[u] = -INFINITY;
#pragma unroll
            for (int j = 0; j < 4; ++j) ov[u][j] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (s >= S) continue;
            const int t0 = tp_range_begin(s, a.n_tiles, S);
            const int t1 = tp_range_begin(s + 1, a.n_tiles, S);
            if (t1 <= t0) continue;
            const long long seg = static_cast<long long>(s) * n_rg + rg;
            lv[u] = a.seg_l[seg * RG + r];
            mv[u] = a.seg_mx[seg * RG + r];
            const float *src = a.seg_O + (seg * RG + r) * a.d;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int dd = 128 * j + 4 * lane;
                if (dd < a.d) ov[u][j] = *reinterpret_cast<const float4 *>(src + dd);
            }
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
            if (s0 + u >= S) break;
            lsum += lv[u];
            mx = fmaxf(mx, mv[u]);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                o[4 * j + 0] += ov[u][j].x;
                o[4 * j + 1] += ov[u][j].y;
                o[4 * j + 2] += ov[u][j].z;
                o[4 * j + 3] += ov[u][j].w;
            }
        }
    }
}

// max over the segments of compacted row k (first segment on ties = lowest slot) and its
// local argmax slot (-1 if the shard has no candidate)
__device__ __forceinline__ void gather_row_max(const CombineArgs &a, int n_rg, int k, float &cmax, int &carg) {
    const int RG = a.rows_per_group;
    const int rg = k / RG, r = k % RG;
    cmax = -INFINITY;
    carg = -1;
    if (a.n_tiles <= 0) return;
    const int S = (a.wide ? a.sc->S_sched : tp_choose_S(n_rg, a.G, a.n_tiles));
    for (int s = 0; s < S; ++s) {
        const int t0 = tp_range_begin(s, a.n_tiles, S);
        const int t1 = tp_range_begin(s + 1, a.n_tiles, S);
        if (t1 <= t0) continue;
        const long long seg = static_cast<long long>(s) * n_rg + rg;
        const float v = a.seg_mx[seg * RG + r];
        if (v > cmax) {
            cmax = v;
            carg = a.seg_arg[seg * RG + r];
        }
    }
}

// dL_cos/dx_hat of an out-of-pool row handled by the main kernel (neg_mode 1 / 2), before
// the factor lambda / N_neg; phi_raw = the shard's unreduced phi partial (sum of hinged
// cosines, or the max cosine).
// R1 fallback (large s): after the fused kernel, an in-pool row whose largest non-target
// exponent fell below REFINE_BELOW (relative to its reference b_r) gets b_r lowered to that
// maximum, and the fused kernel runs again for the batch (R1).  With the exact row
// maximum as the reference no term of the row can underflow or overflow.
constexpr float REFINE_BELOW = -50.f;
__global__ void k_refine_ref(CombineArgs a, float2 *__restrict__ row_ab) {
    const int n_pos = a.sc->n_pos;
    const int n_rg = (a.sc->n_rows + a.rows_per_group - 1) / a.rows_per_group;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n_pos; k += gridDim.x * blockDim.x) {
        float cmax;
        int carg;
        gather_row_max(a, n_rg, k, cmax, carg);
        if (cmax < REFINE_BELOW && cmax > -INFINITY) {
            row_ab[k].y += cmax;
            a.sc_w->refine = 1;
        }
    }
}

__device__ __forceinline__ void neg_row_local(const CombineArgs &a, int n_rg, int kn, float (&g)[16],
                                              float &phi_raw, int &carg) {
    carg = -1;
    if (a.neg_mode == 1) {
        float lsum, mx;
        gather_row_partials(a, n_rg, kn, g, lsum, mx);
        phi_raw = lsum;
    } else {
        float cmax;
        gather_row_max(a, n_rg, kn, cmax, carg);
        phi_raw = cmax;
        zero16(g);
    }
}
// slot c's exact center (lane layout of load_bf16_row), times scale
__device__ __forceinline__ void load_center(const CombineArgs &a, int c, int lane, float scale, float (&v)[16]) {
    if (a.Tc_kind == 1) {
        load_x_row(a.Tc, 1, c, a.d, lane, scale, v);
        return;
    }
    if (a.Tc_kind == 0) {
        load_bf16_row(reinterpret_cast<const __nv_bfloat16 *>(a.Tc) + static_cast<int64_t>(c) * a.d, a.d, lane, scale, v);
        return;
    }
    // K raw rows: fp32 sum over k, then x 1/K (the enqueue's arithmetic, slot_mean16)
    const __nv_bfloat16 *raw = reinterpret_cast<const __nv_bfloat16 *>(a.Tc) + static_cast<int64_t>(c) * a.Kc * a.d;
    float acc[16], r[16];
    zero16(acc);
    for (int k = 0; k < a.Kc; ++k) {
        load_bf16_row(raw + static_cast<int64_t>(k) * a.d, a.d, lane, 1.f, r);
#pragma unroll
        for (int q = 0; q < 16; ++q) acc[q] = __fadd_rn(acc[q], r[q]);
    }
    const float invK = 1.0f / static_cast<float>(a.Kc);
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = __fmul_rn(acc[q], invK) * scale;
}
__device__ __forceinline__ void add_center(const CombineArgs &a, int carg, float coef, float (&g)[16]) {
    const float wc = a.wslot ? a.wslot[carg] : 1.f;
    load_center(a, carg, threadIdx.x & 31, coef * wc, g);
}

// normalisation Jacobian and output: dst = (g - (g . x_hat) x_hat) / ||x||
__device__ __forceinline__ void jacobian(const float (&g)[16], const float (&xh)[16], float inv, float (&out)[16]) {
    float gd = 0.f;
#pragma unroll
    for (int q = 0; q < 16; ++q) gd += g[q] * xh[q];
    gd = warp_sum(gd);
#pragma unroll
    for (int q = 0; q < 16; ++q) out[q] = (g[q] - gd * xh[q]) * inv;
}

// a6: the loss from the per-row terms, by the LAST CTA of the final per-row kernel to finish
// (fixed-order fp64 sums, so deterministic): L_ce = (1/N_pos) sum ell_i, L_cos =
// (1/N_neg) sum phi_i, L = L_ce + lambda L_cos (D11; lambda S:408).
// Replaces a separate one-CTA launch.
__device__ __forceinline__ void loss_tail(const CombineArgs &a, float *loss) {
    __shared__ double sa[256], sb[256];
    __shared__ bool last;
    __syncthreads();  // every row of this CTA has its rowloss written
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&a.sc_w->loss_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int tid = threadIdx.x;
    double ce = 0.0, cs = 0.0;
    for (int64_t i = tid; i < a.N; i += blockDim.x) {
        const double v = __ldcg(a.rowloss + i);
        if (a.comp_idx[i] >= 0) ce += v;
        else cs += v;
    }
    sa[tid] = ce;
    sb[tid] = cs;
    __syncthreads();
    for (int s2 = blockDim.x / 2; s2; s2 >>= 1) {
        if (tid < s2) {
            sa[tid] += sa[tid + s2];
            sb[tid] += sb[tid + s2];
        }
        __syncthreads();
    }
    if (tid == 0) {
        Scalars *sc = a.sc_w;
        const int np = sc->n_pos, nn = sc->n_neg;
        const double Lce = np > 0 ? sa[0] / np : 0.0;
        const double Lcos = nn > 0 ? sb[0] / nn : 0.0;
        const double L = Lce + static_cast<double>(a.lam) * Lcos;
        sc->loss3[0] = L;
        sc->loss3[1] = Lce;
        sc->loss3[2] = Lcos;
        *loss = static_cast<float>(L);
        if (!isfinite(L)) latch(sc, ERR_DEVICE, DET_NONFINITE);
        sc->loss_done = 0u;  // for the next call
    }
}

__device__ __forceinline__ void combine_row(const CombineArgs &a, int64_t i) {
    const int lane = threadIdx.x & 31;
    const int n_pos = a.sc->n_pos, n_neg = a.sc->n_neg;
    const int n_rg = (a.sc->n_rows + a.rows_per_group - 1) / a.rows_per_group;
    const int k = a.comp_idx[i];
    const float inv = a.inv_n[i];
    float xh[16], g[16];
    load_x_row(a.x, a.dtype, i, a.d, lane, inv, xh);
    double row_loss = 0.0;
    if (k >= 0) {
        float o[16], lsum, mx;
        gather_row_partials(a, n_rg, k, o, lsum, mx);
        const double tt = static_cast<double>(a.ttgt[k]);
        const double lr = static_cast<double>(lsum);
        const double et = exp2(tt);
        const double l = lr + et;
        const float2 ab = a.row_ab[k];
        const int ts = a.row_tgt[k];
        const double w = static_cast<double>(a.s) / static_cast<double>(n_pos);
        const float alpha = static_cast<float>(w / l), beta = static_cast<float>(w * (lr / l));
        float Tt[16];
        load_center(a, ts < 0 ? 0 : ts, lane, 1.f, Tt);
#pragma unroll
        for (int q = 0; q < 16; ++q) g[q] = alpha * o[q] - beta * Tt[q];
        const double ell = log1p(lr * exp2(-tt));  // = lse - z_t
        row_loss = ell;
        if (lane == 0) {
            a.st_ell[i] = static_cast<float>(ell);
            a.st_lse[i] = static_cast<float>((static_cast<double>(ab.y) + log2(l)) * 0.6931471805599453);
            a.st_cos[i] = static_cast<float>((tt + a.margin_l2 + ab.y) / (a.s * 1.4426950408889634));
            a.st_phi[i] = 0.f;
            if (!(l > 0.0) || !isfinite(ell) || !(ts >= 0) ||
                (mx < -100.f && static_cast<float>(tt) - mx < 64.f))
                latch(a.sc_w, ERR_DEVICE, (!(ts >= 0) || !isfinite(ell)) ? DET_NONFINITE : DET_UNDERFLOW);
        }
    } else {
        // out-of-pool (L_cos, D10 / NEXT-3): phi = R_c h(cos_c), gradient (lambda/N_neg) dphi
        const float rs = a.phi_mean ? (a.C_occ > 0 ? 1.0f / static_cast<float>(a.C_occ) : 0.f) : 1.f;
        const float w = n_neg > 0 ? a.lam / static_cast<float>(n_neg) : 0.f;
        float phi;
        if (k == -1) {
            // mu path: mu = sum over occupied slots of w_c T_bar_c (kept by the enqueue)
            float mu[16];
            load_mu(a, lane, mu);
            float dot = 0.f;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                g[q] = w * rs * mu[q];
                dot += xh[q] * mu[q];
            }
            dot = warp_sum(dot);
            phi = a.C_occ > 0 ? dot * rs : 0.f;
        } else {
            float raw;
            int carg;
            neg_row_local(a, n_rg, -2 - k, g, raw, carg);
            if (a.neg_mode == 1) {
                phi = a.C_occ > 0 ? raw * rs : 0.f;
#pragma unroll
                for (int q = 0; q < 16; ++q) g[q] *= w * rs;
            } else {
                phi = carg < 0 ? 0.f : (a.hinge ? fmaxf(raw, 0.f) : raw);
                if (carg >= 0 && !(a.hinge && raw <= 0.f)) add_center(a, carg, w, g);
            }
        }
        row_loss = phi;
        if (lane == 0) {
            a.st_phi[i] = phi;
            a.st_ell[i] = 0.f;
            a.st_lse[i] = 0.f;
            a.st_cos[i] = 0.f;
        }
    }
    float out[16];
    jacobian(g, xh, inv, out);
    store_dx_row(a.dx, a.dtype, i, a.d, lane, out);
    if (lane == 0) a.rowloss[i] = row_loss;
}

__global__ void __launch_bounds__(256, 2) k_combine(CombineArgs a, float *loss) {
    clear_hash_slice(a, gridDim.x);
    const int64_t i = static_cast<int64_t>(blockIdx.x) * CB_ROWS + (threadIdx.x >> 5);
    if (i < a.N) combine_row(a, i);
    loss_tail(a, loss);
}

// ------------------------------------------------------------------ multi-rank combine
// Per global row i, this rank's partial of the softmax statistics over its slot shard:
//   in-pool rows:     (l_rest_r, max_r, ttgt_r, b_r)  (ttgt_r = -inf unless rank r owns t_i)
//   out-of-pool rows: (phi_r, 0, 0, 0)               phi_r = x_hat_i . mu_r (unreduced)
// These are all-gathered (C3); every rank then finalises identically (k_finalize_multi).
__global__ void __launch_bounds__(256, 2) k_local_rows(CombineArgs a, float4 *__restrict__ scal) {
    const int lane = threadIdx.x & 31;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * CB_ROWS + (threadIdx.x >> 5);
    if (i >= a.N) return;
    const int n_rg = (a.sc->n_rows + a.rows_per_group - 1) / a.rows_per_group;
    const int k = a.comp_idx[i];
    if (k >= 0) {
        // (only the scalars: l_rest and max over the segments)
        const int RG = a.rows_per_group;
        const int rg = k / RG, r = k % RG;
        float lsum = 0.f, mx = -INFINITY;
        if (a.n_tiles > 0) {
            const int S = (a.wide ? a.sc->S_sched : tp_choose_S(n_rg, a.G, a.n_tiles));
            for (int s = lane; s < S; s += 32) {  // lanes split the segments, fixed-order tree below
                const int t0 = tp_range_begin(s, a.n_tiles, S);
                const int t1 = tp_range_begin(s + 1, a.n_tiles, S);
                if (t1 <= t0) continue;
                const long long seg = static_cast<long long>(s) * n_rg + rg;
                lsum += a.seg_l[seg * RG + r];
                mx = fmaxf(mx, a.seg_mx[seg * RG + r]);
            }
        }
        lsum = warp_sum(lsum);
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0) scal[i] = make_float4(lsum, mx, a.ttgt[k], a.row_ab[k].y);
    } else if (k <= -2) {
        float g[16], raw;
        int carg;
        neg_row_local(a, n_rg, -2 - k, g, raw, carg);
        if (lane == 0) scal[i] = make_float4(raw, 0.f, 0.f, 0.f);
    } else {
        float mu[16], xh[16];
        load_mu(a, lane, mu);
        load_x_row(a.x, a.dtype, i, a.d, lane, a.inv_n[i], xh);
        float dot = 0.f;
#pragma unroll
        for (int q = 0; q < 16; ++q) dot += xh[q] * mu[q];
        dot = warp_sum(dot);
        if (lane == 0) scal[i] = make_float4(dot, 0.f, 0.f, 0.f);  // x_hat . mu_r (unreduced)
    }
}

// Global finalisation from the gathered partials (rank order => deterministic), and this
// rank's LINEAR share of dL/dx (projection applied), summed over ranks by the
// reduce-scatter (C4):
//   in-pool:     g_r = (s/N_pos) (O_r / l - [r owns t] (l_rest / l) T_t)
//   out-of-pool: g_r = mu_r / (N_neg C_occ)
__device__ __forceinline__ void finalize_row(const CombineArgs &a, const float4 *__restrict__ scal_all, int W,
                                             int64_t N, float *__restrict__ dx_part, int64_t i) {
    const int lane = threadIdx.x & 31;
    const int n_pos = a.sc->n_pos, n_neg = a.sc->n_neg;
    const int n_rg = (a.sc->n_rows + a.rows_per_group - 1) / a.rows_per_group;
    const int k = a.comp_idx[i];
    const float inv = a.inv_n[i];
    float xh[16], g[16];
    load_x_row(a.x, a.dtype, i, a.d, lane, inv, xh);
    double row_loss = 0.0;
    if (k >= 0) {
        // every shard used its own reference b_r: rescale to the common B* = max_r b_r
        float Bs = -INFINITY;
        for (int r = 0; r < W; ++r) Bs = fmaxf(Bs, scal_all[static_cast<int64_t>(r) * N + i].w);
        double lr = 0.0;
        float mx = -INFINITY, tt = -INFINITY;
        for (int r = 0; r < W; ++r) {
            const float4 v = scal_all[static_cast<int64_t>(r) * N + i];
            lr += static_cast<double>(v.x) * exp2(static_cast<double>(v.w) - Bs);
            mx = fmaxf(mx, v.y + (v.w - Bs));
            tt = fmaxf(tt, v.z + (v.w - Bs));
        }
        float o[16], lsum, mxl;
        gather_row_partials(a, n_rg, k, o, lsum, mxl);
        const double l = lr + exp2(static_cast<double>(tt));
        const double w = static_cast<double>(a.s) / static_cast<double>(n_pos);
        const int ts = a.row_tgt[k];  // >= 0 iff this rank owns the target slot
        const float my_scale = static_cast<float>(exp2(static_cast<double>(a.row_ab[k].y) - Bs));
        const float alpha = static_cast<float>(w / l) * my_scale;
        const float beta = ts >= 0 ? static_cast<float>(w * (lr / l)) : 0.f;
        float Tt[16];
        load_center(a, ts < 0 ? 0 : ts, lane, 1.f, Tt);
#pragma unroll
        for (int q = 0; q < 16; ++q) g[q] = alpha * o[q] - beta * Tt[q];
        const double ell = log1p(lr * exp2(-static_cast<double>(tt)));
        row_loss = ell;
        if (lane == 0) {
            a.st_ell[i] = static_cast<float>(ell);
            a.st_lse[i] = static_cast<float>((static_cast<double>(Bs) + log2(l)) * 0.6931471805599453);
            a.st_cos[i] = static_cast<float>((static_cast<double>(tt) + a.margin_l2 + Bs) / (a.s * 1.4426950408889634));
            a.st_phi[i] = 0.f;
            if (!(l > 0.0) || !isfinite(ell) || (mx < -100.f && tt - mx < 64.f))
                latch(a.sc_w, ERR_DEVICE, !isfinite(ell) ? DET_NONFINITE : DET_UNDERFLOW);
        }
    } else {
        const float rs = a.phi_mean ? (a.C_occ > 0 ? 1.0f / static_cast<float>(a.C_occ) : 0.f) : 1.f;
        const float w = n_neg > 0 ? a.lam / static_cast<float>(n_neg) : 0.f;
        double phi = 0.0;
        if (a.neg_mode == 2 && k <= -2) {
            // hardest negative: global max over the shards (first rank = lowest slot on ties);
            // only the owning shard contributes the gradient T_bar_c* / ||T_bar_c*||
            float gmax = -INFINITY;
            int rw = -1;
            for (int r = 0; r < W; ++r) {
                const float v = scal_all[static_cast<int64_t>(r) * N + i].x;
                if (v > gmax) { gmax = v; rw = r; }
            }
            phi = rw < 0 ? 0.0 : static_cast<double>(a.hinge ? fmaxf(gmax, 0.f) : gmax);
            float raw;
            int carg;
            neg_row_local(a, n_rg, -2 - k, g, raw, carg);
            if (rw == a.my_rank && carg >= 0 && !(a.hinge && gmax <= 0.f)) add_center(a, carg, w, g);
        } else {
            if (k <= -2) {
                float raw;
                int carg;
                neg_row_local(a, n_rg, -2 - k, g, raw, carg);
            } else {
                load_mu(a, lane, g);
            }
#pragma unroll
            for (int q = 0; q < 16; ++q) g[q] *= w * rs;
            for (int r = 0; r < W; ++r) phi += static_cast<double>(scal_all[static_cast<int64_t>(r) * N + i].x);
            phi = a.C_occ > 0 ? phi * rs : 0.0;
        }
        row_loss = phi;
        if (lane == 0) {
            a.st_phi[i] = static_cast<float>(phi);
            a.st_ell[i] = 0.f;
            a.st_lse[i] = 0.f;
            a.st_cos[i] = 0.f;
        }
    }
    float out[16];
    jacobian(g, xh, inv, out);
    float *dst = dx_part + i * a.d;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int dd = 128 * j + 4 * lane;
        if (dd < a.d) *reinterpret_cast<float4 *>(dst + dd) = make_float4(out[4 * j], out[4 * j + 1], out[4 * j + 2], out[4 * j + 3]);
    }
    if (lane == 0) a.rowloss[i] = row_loss;
}

__global__ void __launch_bounds__(256, 2) k_finalize_multi(CombineArgs a, const float4 *__restrict__ scal_all,
                                                        int W, int64_t N, float *__restrict__ dx_part, float *loss) {
    clear_hash_slice(a, gridDim.x);
    const int64_t i = static_cast<int64_t>(blockIdx.x) * CB_ROWS + (threadIdx.x >> 5);
    if (i < N) finalize_row(a, scal_all, W, N, dx_part, i);
    loss_tail(a, loss);
}

// fp32 -> bf16 (the multi-rank dx output; the bf16 shadow of an fp32 pool after set_state)
__global__ void k_cast_bf16(const float *__restrict__ src, __nv_bfloat16 *__restrict__ dst, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        dst[i] = __float2bfloat16_rn(src[i]);
}

// emulated-world collectives (one device): fixed rank order
__global__ void k_max_i64_into(int64_t *__restrict__ acc, const int64_t *__restrict__ src, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (src[i] > acc[i]) acc[i] = src[i];
}
__global__ void k_add_f32_into(float *__restrict__ acc, const float *__restrict__ src, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        acc[i] += src[i];
}
// pack (tseq, tmax bits) for the MAX all-reduce (C2)
__global__ void k_pack_tseq(const int64_t *__restrict__ tseq, const Scalars *__restrict__ sc, int64_t N,
                            int64_t *__restrict__ ext) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i <= N;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        ext[i] = i < N ? tseq[i] : static_cast<int64_t>(sc->tmax_bits);
}
__global__ void k_unpack_tseq(const int64_t *__restrict__ ext, int64_t N, int64_t *__restrict__ tseq,
                              int *__restrict__ tmax_glob) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i <= N;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (i < N) tseq[i] = ext[i];
        else *tmax_glob = static_cast<int>(ext[N]);
    }
}


}  // namespace f2c
