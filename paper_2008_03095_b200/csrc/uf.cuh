// uf.cuh -- concurrent union-find over one lane of the label matrix.
//
// Every lane r is an independent sampled graph; its forest lives in column r
// of L.  Cells are either ROOT|count (bit 31 set) or a parent pointer to a
// strictly smaller id, so the root of every tree is its minimum vertex id --
// exactly the min-id label the reference's propagation converges to (SURVEY
// S6, propagation.py:1-8).  All accesses go through L2 (relaxed, gpu scope).
#pragma once
#include "common.cuh"

namespace imx {

constexpr uint32_t ROOT = 0x80000000u;
constexpr uint32_t COUNT = 0x7FFFFFFFu;

// Layout of a label matrix.  Rows (the default): cell (v, r) at v * ld + r,
// simulation-contiguous (propagation.py:1-8).  Lane tiles (very wide
// contexts, ctx.cu): tiles of tl = 2^tsh lanes, each tile a contiguous
// [n][tl] block, so the walks of one tile's compression stay in L2 without a
// copy: cell (v, r) at (r >> tsh) * tstride + v * tl + (r & tmask).  An
// int64 row length converts to the row layout, so code that only ever sees
// rows keeps passing ld.
struct Lay {
    int64_t ld;          // cells per contiguous row run: the row, or tl
    int64_t tstride;     // cells per tile (0: rows)
    int tsh;             // tile of lane r = r >> tsh (31: rows)
    uint32_t tmask;
    __host__ __device__ Lay(int64_t row_ld = 0) : ld(row_ld), tstride(0), tsh(31), tmask(0x7fffffffu) {}
    __host__ __device__ static Lay tiles(int64_t n, int shift) {
        Lay y((int64_t)1 << shift);
        y.tstride = n << shift;
        y.tsh = shift;
        y.tmask = (1u << shift) - 1u;
        return y;
    }
    __host__ __device__ bool tiled() const { return tstride != 0; }
    __host__ __device__ int64_t off(int64_t v, int r) const {
        return (int64_t)(r >> tsh) * tstride + v * ld + (int64_t)(r & tmask);
    }
};

// quad q (lanes 4q..4q+3) of row v; rows keep the plain row-pointer form
__device__ __forceinline__ uint4 row_quad(const uint32_t *L, const Lay &y, int64_t v, int q) {
    if (!y.tiled()) return reinterpret_cast<const uint4 *>(L + v * y.ld)[q];
    return *reinterpret_cast<const uint4 *>(L + y.off(v, q << 2));
}
__device__ __forceinline__ int64_t cell_off(const Lay &y, int64_t v, int r) {
    return y.tiled() ? y.off(v, r) : v * y.ld + r;
}

__device__ __forceinline__ uint32_t *cell(uint32_t *L, const Lay &y, uint32_t v, int r) {
    return L + y.off(v, r);
}
__device__ __forceinline__ const uint32_t *cell(const uint32_t *L, const Lay &y, uint32_t v, int r) {
    return L + y.off(v, r);
}
__device__ __forceinline__ bool is_root(uint32_t w) { return (w & ROOT) != 0; }
// label of vertex v from its (compressed) cell word
__device__ __forceinline__ uint32_t label_of(uint32_t v, uint32_t w) { return is_root(w) ? v : w; }

// Hub cells during hooking.  On skewed graphs the lowest ids are the hubs
// and the roots of the giant components, so every union in those
// components ends at the same few cells of a lane: one L2 sector serialises
// them.  Vertex 0 is a root in every lane (nothing is smaller), so its cell
// is never read; the other hub ids below kHotHook are read through L1.  A
// stale word is safe: a stale ROOT only makes a union link under, or
// compare against, a node that is no longer a root but still has a smaller
// id than what is linked under it (the tree stays min-rooted and the CAS on
// a stale root fails and reports its parent); a stale parent is an ancestor.
#ifndef IMX_HOT_HOOK
#define IMX_HOT_HOOK 4
#endif
constexpr uint32_t kHotHook = IMX_HOT_HOOK;

__device__ __forceinline__ uint32_t ld_hook(uint32_t *L, const Lay &ld, uint32_t v, int r) {
    if (kHotHook > 0 && v < kHotHook) {
        if (v == 0) return ROOT;
        uint32_t w;
        asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(w) : "l"(cell(L, ld, v, r)));
        return w;
    }
    return ld_relaxed(cell(L, ld, v, r));
}

// Two root searches advanced in lock step so their loads overlap.  Path
// splitting: every visited node is re-pointed at its grandparent (benign
// races -- any value ever stored in a cell is an ancestor in the same tree).
// On entry wa = L[xa], wb = L[xb]; on exit xa, xb are roots.
__device__ __forceinline__ void find2(uint32_t *L, const Lay &ld, int r, uint32_t &xa, uint32_t wa,
                                      uint32_t &xb, uint32_t wb) {
    for (;;) {
        const bool da = is_root(wa), db = is_root(wb);
        if (da && db) return;
        uint32_t ga = 0, gb = 0;
        if (!da) ga = ld_hook(L, ld, wa, r);
        if (!db) gb = ld_hook(L, ld, wb, r);
        if (!da) {
            if (!is_root(ga)) st_relaxed(cell(L, ld, xa, r), ga);
            xa = wa;
            wa = ga;
        }
        if (!db) {
            if (!is_root(gb)) st_relaxed(cell(L, ld, xb, r), gb);
            xb = wb;
            wb = gb;
        }
    }
}

// Union of a and b in lane r: CAS-hook the larger root under the smaller.
// During hooking every root cell is exactly ROOT (member counts are only
// written by the compress pass).  Returns 1 when a hook happened.
__device__ __forceinline__ int unite(uint32_t *L, const Lay &ld, uint32_t a, uint32_t b, int r) {
    uint32_t wa = ld_hook(L, ld, a, r);
    uint32_t wb = ld_hook(L, ld, b, r);
    find2(L, ld, r, a, wa, b, wb);
    while (a != b) {
        const uint32_t lo = a < b ? a : b, hi = a < b ? b : a;
        const uint32_t old = atomicCAS(cell(L, ld, hi, r), ROOT, lo);
        if (old == ROOT) return 1;
        a = lo;
        b = hi;
        find2(L, ld, r, a, ld_hook(L, ld, lo, r), b, old);
    }
    return 0;
}

// Root of x given its parent p (p = L[x], not a root word); re-points each
// visited node at its grandparent with atomicMin, so it is safe against the
// owners' final stores of the root (the smallest id of the tree).
__device__ __forceinline__ uint32_t find_split(uint32_t *L, const Lay &ld, uint32_t x, uint32_t p, int r) {
    for (;;) {
        const uint32_t gw = ld_relaxed(cell(L, ld, p, r));
        if (is_root(gw)) return p;
        atomicMin(cell(L, ld, x, r), gw);
        x = p;
        p = gw;
    }
}

}  // namespace imx
