// k_merge.cu -- X4 of the z-slab sharded path on the device: the cross-slab label merge that every
// rank runs identically on the all-gathered boundary tables (it replaces, at volume
// scale, the paper's single-image largest-contour step P:283-285).
//
// Input: G blocks (one per rank, in rank order) of roix_merge_block_words(pair_cap, root_cap)
// uint64 words: [npairs, nroots, pairs (2 pair_cap), labels (root_cap), sizes (root_cap)].  A rank's
// labels are the global minimum indices of its components touching a slab face, ascending; every
// rank's labels lie inside its own slab's index range, so the blocks concatenate in ascending order.
// A pair (a, b) says the components labelled a and b are one (they overlap across a slab face).
// Output: the map -- every boundary label, its merged label (the minimum label of its merged
// component: union by minimum, so the result does not depend on the pair order, G-14) and the merged
// component's total size -- and its length (device).
#include "common.cuh"
#include "kernels.cuh"

namespace roix {

struct MergeWS {
    uint32_t *parent;   // [G root_cap]
    uint64_t *tot;      // [G root_cap]
    uint64_t *off;      // [G + 1]
};

static size_t mg_carve(void *base, uint32_t G, uint64_t root_cap, MergeWS *w) {
    auto al = [](size_t v) { return (v + 255) & ~(size_t)255; };
    const uint64_t M = (uint64_t)G * root_cap;
    const size_t a = al(M * 4 + 4), b = al(M * 8 + 8), c = al((G + 1) * 8);
    if (w) {
        char *p = (char *)base;
        w->parent = (uint32_t *)p;
        w->tot = (uint64_t *)(p + a);
        w->off = (uint64_t *)(p + a + b);
    }
    return a + b + c;
}

struct Blocks {
    const uint64_t *g;
    uint64_t pair_cap, root_cap, words;   // words per block
    uint32_t G;
    __device__ uint64_t npairs(uint32_t r) const { return min(g[r * words], pair_cap); }
    __device__ uint64_t nroots(uint32_t r) const { return min(g[r * words + 1], root_cap); }
    __device__ const uint64_t *pairs(uint32_t r) const { return g + r * words + 2; }
    __device__ const uint64_t *labels(uint32_t r) const { return g + r * words + 2 + 2 * pair_cap; }
    __device__ const uint64_t *sizes(uint32_t r) const { return g + r * words + 2 + 2 * pair_cap + root_cap; }
};

__device__ __forceinline__ uint32_t mg_find(uint32_t *parent, uint32_t x) {
    uint32_t p = parent[x];
    while (p != x) {   // path halving: pointers only move to ancestors, so racing writes stay valid
        const uint32_t gp = parent[p];
        if (gp != p) atomicMin(&parent[x], gp);
        x = p;
        p = gp;
    }
    return x;
}

__device__ void mg_unite(uint32_t *parent, uint32_t a, uint32_t b) {
    while (true) {
        a = mg_find(parent, a);
        b = mg_find(parent, b);
        if (a == b) return;
        if (a < b) {
            const uint32_t t = a;
            a = b;
            b = t;
        }
        const uint32_t old = atomicMin(&parent[a], b);   // the larger root under the smaller
        if (old == a) return;
        a = old;
    }
}

// rank offsets of the concatenated tables, the map length, capacity checks (one warp)
__global__ void k_merge_prep(Blocks B, MergeWS w, uint64_t *nmap, roix_scalars *sc) {
    if (threadIdx.x != 0) return;
    uint64_t off = 0;
    uint32_t bad = 0;
    for (uint32_t r = 0; r < B.G; r++) {
        w.off[r] = off;
        off += B.nroots(r);
        bad |= B.g[r * B.words] > B.pair_cap || B.g[r * B.words + 1] > B.root_cap;
    }
    w.off[B.G] = off;
    *nmap = off;
    if (bad) set_err(sc, ROIX_ERR_CAPACITY);
}

__global__ void k_merge_build(Blocks B, MergeWS w, uint64_t *map_label, uint64_t *map_total) {
    const uint64_t total = (uint64_t)B.G * B.root_cap;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = (uint32_t)(t / B.root_cap);
        const uint64_t k = t % B.root_cap;
        if (k >= B.nroots(r)) continue;
        const uint64_t i = w.off[r] + k;
        map_label[i] = B.labels(r)[k];
        map_total[i] = B.sizes(r)[k];   // the label's own size until k_merge_final
        w.parent[i] = (uint32_t)i;
        w.tot[i] = 0;
    }
}

__device__ __forceinline__ int64_t mg_index(const uint64_t *L, uint64_t m, uint64_t lab) {
    uint64_t lo = 0, hi = m;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (L[mid] < lab) lo = mid + 1;
        else hi = mid;
    }
    return (lo < m && L[lo] == lab) ? (int64_t)lo : -1;
}

__global__ void k_merge_union(Blocks B, MergeWS w, const uint64_t *map_label, const uint64_t *nmap, roix_scalars *sc) {
    const uint64_t m = *nmap;
    const uint64_t total = (uint64_t)B.G * B.pair_cap;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = (uint32_t)(t / B.pair_cap);
        const uint64_t k = t % B.pair_cap;
        if (k >= B.npairs(r)) continue;
        const int64_t a = mg_index(map_label, m, B.pairs(r)[2 * k]), b = mg_index(map_label, m, B.pairs(r)[2 * k + 1]);
        if (a < 0 || b < 0) {   // a pair naming a label missing from the tables: malformed input
            set_err(sc, ROIX_ERR_FORMAT);
            continue;
        }
        mg_unite(w.parent, (uint32_t)a, (uint32_t)b);
    }
}

// roots: flatten, and sum every label's size into its root
__global__ void k_merge_flatten(MergeWS w, const uint64_t *map_total, const uint64_t *nmap) {
    const uint64_t m = *nmap;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = mg_find(w.parent, (uint32_t)i);
        atomicAdd((unsigned long long *)&w.tot[r], (unsigned long long)map_total[i]);
    }
}

__global__ void k_merge_final(MergeWS w, const uint64_t *map_label, uint64_t *map_final, uint64_t *map_total,
                              const uint64_t *nmap) {
    const uint64_t m = *nmap;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = mg_find(w.parent, (uint32_t)i);
        map_final[i] = map_label[r];
        map_total[i] = w.tot[r];
    }
}

}  // namespace roix

using namespace roix;

size_t merge_workspace_bytes(uint32_t G, uint64_t root_cap) { return mg_carve(nullptr, G, root_cap, nullptr); }

cudaError_t launch_merge(const uint64_t *gathered, uint32_t G, uint64_t pair_cap, uint64_t root_cap,
                         uint64_t *map_label, uint64_t *map_final, uint64_t *map_total, uint64_t *nmap, void *ws,
                         roix_scalars *sc, cudaStream_t st) {
    MergeWS w;
    mg_carve(ws, G, root_cap, &w);
    Blocks B;
    B.g = gathered;
    B.pair_cap = pair_cap;
    B.root_cap = root_cap;
    B.words = 2 + 2 * pair_cap + 2 * root_cap;
    B.G = G;
    auto grid = [](uint64_t work) {
        uint64_t b = (work + 255) / 256;
        const uint64_t cap = (uint64_t)num_sms() * 4;
        return (unsigned)(b < 1 ? 1 : b < cap ? b : cap);
    };
    k_merge_prep<<<1, 32, 0, st>>>(B, w, nmap, sc);
    k_merge_build<<<grid((uint64_t)G * root_cap), 256, 0, st>>>(B, w, map_label, map_total);
    k_merge_union<<<grid((uint64_t)G * pair_cap), 256, 0, st>>>(B, w, map_label, nmap, sc);
    k_merge_flatten<<<grid((uint64_t)G * root_cap), 256, 0, st>>>(w, map_total, nmap);
    k_merge_final<<<grid((uint64_t)G * root_cap), 256, 0, st>>>(w, map_label, map_final, map_total, nmap);
    return cudaGetLastError();
}
