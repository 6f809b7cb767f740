// Register-resident Walsh-Hadamard transform of 1024-element (or smaller)
// blocks by one warp, with the reference's exact radix-2 network
// (_fast.pyx:23-41: stages h = 1, 2, 4, ...; butterfly (a+b, a-b)).
//
// A block of PAD = 32*E doubles lives in shared memory under the swizzle
// sw(j) = (j & ~31) | ((j & 31) ^ ((j >> 5) & 15)) (at most the minimal 2
// wavefronts per 8-byte access for both access patterns below).  Layout A: lane l holds j = l*E + e (stages h < E in
// registers); layout B: lane l holds j = e*32 + l (stages E <= h < 32 by
// shfl_xor, h >= 32 in registers).  Every output is produced by the same
// tree of fp64 add/sub as the reference's loop nest, so results are bit
// identical.
#pragma once
#include "common.cuh"

namespace srlu {

// XOR the lane bits with bits 5..8 only: block-local for any block >= 512
__device__ __forceinline__ int fwht_sw(int j) { return (j & ~31) | ((j & 31) ^ ((j >> 5) & 15)); }

template <int E>
__device__ __forceinline__ void fwht_block_warp(double *blk, int lane) {
    static_assert(E >= 1 && E <= 32 && (E & (E - 1)) == 0, "E must be a power of two <= 32");
    double v[E];
    // layout A
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = blk[fwht_sw(lane * E + e)];
#pragma unroll
    for (int h = 1; h < E; h <<= 1) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if ((e & h) == 0) {
                const double a = v[e], b = v[e + h];
                v[e] = __dadd_rn(a, b);
                v[e + h] = __dsub_rn(a, b);
            }
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) blk[fwht_sw(lane * E + e)] = v[e];
    __syncwarp();
    // layout B
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = blk[fwht_sw(e * 32 + lane)];
#pragma unroll
    for (int h = E; h < 32; h <<= 1) {
        const bool up = (lane & h) != 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const double p = __shfl_xor_sync(0xffffffffu, v[e], h);
            v[e] = up ? __dsub_rn(p, v[e]) : __dadd_rn(v[e], p);
        }
    }
#pragma unroll
    for (int hh = 1; hh < E; hh <<= 1) {  // h = 32*hh
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if ((e & hh) == 0) {
                const double a = v[e], b = v[e + hh];
                v[e] = __dadd_rn(a, b);
                v[e + hh] = __dsub_rn(a, b);
            }
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) blk[fwht_sw(e * 32 + lane)] = v[e];
    __syncwarp();
}

// Stages h = 1..16 of one value per lane (index j = 32*q + lane): the
// reference's butterflies (a + b, a - b), lower index first, via shuffles.
// Lower lane: v + p; upper lane: p - v.  Both are fma(s, v, p) with
// s = +-1 (the product is exact, one rounding: bit-identical to the add).
__device__ __forceinline__ double pm_one(bool neg) {
    return __hiloint2double(neg ? (int)0xBFF00000 : 0x3FF00000, 0);
}

__device__ __forceinline__ double fwht_lane_stages(double v, int lane) {
#pragma unroll
    for (int h = 1; h < 32; h <<= 1) {
        const double p = __shfl_xor_sync(0xffffffffu, v, h);
        v = __fma_rn(pm_one(lane & h), v, p);
    }
    return v;
}

// The remaining stages h = 32 .. 16*E of a 32*E block whose stages h < 32
// were already applied (fwht_lane_stages): layout B, registers only.
template <int E>
__device__ __forceinline__ void fwht_block_warp_hi(double *blk, int lane) {
    double v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = blk[fwht_sw(e * 32 + lane)];
#pragma unroll
    for (int hh = 1; hh < E; hh <<= 1) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if ((e & hh) == 0) {
                const double a = v[e], b = v[e + hh];
                v[e] = __dadd_rn(a, b);
                v[e + hh] = __dsub_rn(a, b);
            }
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) blk[fwht_sw(e * 32 + lane)] = v[e];
    __syncwarp();
}

__device__ __forceinline__ void fwht_block_warp_hi_dyn512(double *blk, int bsize, int lane) {
    switch (bsize) {
        case 512: fwht_block_warp_hi<16>(blk, lane); break;
        case 256: fwht_block_warp_hi<8>(blk, lane); break;
        case 128: fwht_block_warp_hi<4>(blk, lane); break;
        case 64: fwht_block_warp_hi<2>(blk, lane); break;
        default: break;  // 32: nothing left
    }
}

// dispatch on the block length (32 <= pad <= 1024, power of two)
__device__ __forceinline__ void fwht_block_warp_dyn(double *blk, int pad, int lane) {
    switch (pad) {
        case 1024: fwht_block_warp<32>(blk, lane); break;
        case 512: fwht_block_warp<16>(blk, lane); break;
        case 256: fwht_block_warp<8>(blk, lane); break;
        case 128: fwht_block_warp<4>(blk, lane); break;
        case 64: fwht_block_warp<2>(blk, lane); break;
        default: fwht_block_warp<1>(blk, lane); break;
    }
}

// same for blocks of at most 512 points (16 registers per lane)
__device__ __forceinline__ void fwht_block_warp_dyn512(double *blk, int pad, int lane) {
    switch (pad) {
        case 512: fwht_block_warp<16>(blk, lane); break;
        case 256: fwht_block_warp<8>(blk, lane); break;
        case 128: fwht_block_warp<4>(blk, lane); break;
        case 64: fwht_block_warp<2>(blk, lane); break;
        default: fwht_block_warp<1>(blk, lane); break;
    }
}

// Output-pruned cross-block stages: the value at block B, in-block offset
// o (swizzled) of the full transform whose NB blocks (stride bsize) were
// transformed in place.  Only the NB-1 butterfly nodes feeding that output
// are formed, level by level (stage h = bsize first), with exactly the
// operands and order of the full network (bit-identical).
// Blocks b >= nzb are all-zero and not stored (x + 0 and 0 +- x are exact).
template <int NB>
__device__ __forceinline__ double wht_pick(const double *row, int bsize, int o, int B, int nzb = NB) {
    double u[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) u[b] = b < nzb ? row[b * bsize + o] : 0.0;
#pragma unroll
    for (int s = 1, lvl = 0; s < NB; s <<= 1, ++lvl) {
        const double sg = pm_one((B >> lvl) & 1);
#pragma unroll
        for (int i = 0; i < NB / (2 * s); ++i) u[i] = __fma_rn(sg, u[2 * i + 1], u[2 * i]);
    }
    return u[0];
}

// Value at output index q of the full pad-point transform whose bsize-point
// blocks (nb = pad/bsize <= 16 of them, swizzled) were transformed in
// place: the remaining stages h = bsize, 2*bsize, ... combine the blocks at
// offset q % bsize in the reference's order (output-pruned, wht_pick).
// Blocks b >= nzb are not stored (all zero).
__device__ __forceinline__ double fwht_combine_blocks(const double *row, int bsize, int nb, int q,
                                                      int nzb = 16) {
    const int o = fwht_sw(q & (bsize - 1)), B = q / bsize;
    switch (nb) {
        case 1: return row[o];
        case 2: return wht_pick<2>(row, bsize, o, B, nzb);
        case 4: return wht_pick<4>(row, bsize, o, B, nzb);
        case 8: return wht_pick<8>(row, bsize, o, B, nzb);
        default: return wht_pick<16>(row, bsize, o, B, nzb);
    }
}

}  // namespace srlu
