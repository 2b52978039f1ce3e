// sa_tree.cu -- the paper's contrastive workload: a flattened suffix tree
// searched on the GPU, results normalised to SA intervals (Sec. III: "the suffix tree
// can be transmitted into flatten tree consisting of an array of edges"; Table V STK).
//
// The tree is derived from the index's suffix array: its internal nodes are the lcp-intervals of the
// SA (an lcp-interval l-[i..j] is a maximal SA range whose suffixes share exactly l leading bases,
// l = string depth), children are split by the base at depth l, leaves are single SA ranks.
//   * LCP[r] = lcp(S_SA[r-1], S_SA[r]) on the GPU (32 bases per compare step);
//   * the lcp-interval tree by the bottom-up stack traversal of the LCP array (host, O(n));
//   * nodes flattened into 32-byte records {lb, rb, depth, SA[lb], child[a,c,g,t]} (child = node id,
//     or 0x80000000 | SA rank for a leaf, or 0xFFFFFFFF for none) -- one sector per node;
//   * search: one thread per read walks from the root, one node and one edge-label compare per
//     branching level (the paper's O(m) walk).  A failed walk yields the insertion point, so
//     every read gets exactly the SA search's [lo, hi).
#include <algorithm>
#include <new>
#include <vector>

#include "sa_search.cuh"

struct sa_tree {
    const sa_index *idx = nullptr;  // borrowed: the tree reads the index's text and SA
    uint64_t nodes = 0;
    uint32_t root = 0;
    uint4 *node = nullptr;          // dev: 2 uint4 per node
    uint64_t device_bytes = 0;
};

namespace {

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint32_t kLeaf = 0x80000000u;

__global__ void k_lcp(const uint64_t *__restrict__ text, uint64_t n, const uint32_t *__restrict__ sa, uint32_t stride,
                      uint32_t *__restrict__ lcp) {
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (uint64_t)gridDim.x * blockDim.x) {
        if (r == 0) { lcp[0] = 0; continue; }
        const uint64_t a = sa[(r - 1) * stride], b = sa[r * stride];
        const uint64_t la = n - a, lb = n - b, lmax = la < lb ? la : lb;
        uint64_t l = 0;
        while (l < lmax) {
            const uint64_t x = text_window(text, a + l) ^ text_window(text, b + l);
            const uint64_t rem = lmax - l;
            if (x) {
                const uint64_t d = (uint64_t)(__clzll((long long)x) >> 1);
                l += d < rem ? d : rem;
                break;
            }
            l += rem < 32 ? rem : 32;
        }
        lcp[r] = (uint32_t)l;
    }
}

struct Frame {
    uint32_t lcp, lb;
    uint32_t first_child = kNone, last_child = kNone;  // internal children, in SA order
};

struct HostTree {
    std::vector<uint32_t> lb, rb, depth, pos, sib;
    std::vector<uint32_t> child;  // 4 per node
};

// base at depth d of suffix s (0..3), or 4 when the suffix has exactly d bases
inline uint32_t base_at(const std::vector<uint64_t> &text, uint64_t n, uint64_t s, uint64_t d) {
    const uint64_t i = s + d;
    if (i >= n) return 4;
    return (uint32_t)((text[i >> 5] >> (62 - 2 * (i & 31))) & 3u);
}

uint32_t new_node(HostTree &t, uint32_t lb, uint32_t rb, uint32_t depth, const std::vector<uint32_t> &sa) {
    const uint32_t id = (uint32_t)t.lb.size();
    t.lb.push_back(lb);
    t.rb.push_back(rb);
    t.depth.push_back(depth);
    t.pos.push_back(sa[lb]);
    t.sib.push_back(kNone);
    for (int c = 0; c < 4; ++c) t.child.push_back(kNone);
    return id;
}

// children of node v: its internal child intervals and the single-rank leaves between them
void fill_children(HostTree &t, uint32_t v, uint32_t first_child, const std::vector<uint32_t> &sa,
                   const std::vector<uint64_t> &text, uint64_t n) {
    const uint32_t lb = t.lb[v], rb = t.rb[v], d = t.depth[v];
    uint32_t ch = first_child;
    uint64_t x = lb;
    while (x <= rb) {
        uint32_t target, start;
        if (ch != kNone && t.lb[ch] == x) {
            target = ch;
            start = (uint32_t)x;
            x = (uint64_t)t.rb[ch] + 1;
            ch = t.sib[ch];
        } else {
            target = kLeaf | (uint32_t)x;
            start = (uint32_t)x;
            x += 1;
        }
        const uint32_t c = base_at(text, n, sa[start], d);
        if (c < 4) t.child[4ull * v + c] = target;  // c == 4: the suffix of exactly d bases (sorts first, at lb)
    }
}

}  // namespace

extern "C" sa_status sa_tree_create(const sa_index *idx, sa_tree **out) {
    sa_clear_error();
    if (!idx || !out) { sa_set_error("NULL argument"); return SA_EINVAL; }
    *out = nullptr;
    const uint64_t n = idx->n;
    if (idx->nparts > 1) { sa_set_error("the tree needs a whole index, not a partition"); return SA_EINVAL; }
    if (n >= 0x7FFFFFFFull) { sa_set_error("the flattened tree needs n < 2^31 (leaf tag bit)"); return SA_ETOOLONG; }
    SA_CUDA_TRY(cudaSetDevice(idx->device));
    // ---- LCP on the GPU ----
    const SaView v = sa_view(idx);
    std::vector<uint32_t> lcp(n + 1), sa(n);
    {
        DevBuf<uint32_t> d_lcp;
        SA_TRY(d_lcp.alloc(n, nullptr, "lcp"));
        uint64_t blocks = (n + 255) / 256;
        if (blocks > 148ull * 64) blocks = 148ull * 64;
        k_lcp<<<(unsigned)blocks, 256>>>(idx->text, n, v.base, v.stride, d_lcp.p);
        SA_CUDA_TRY(cudaGetLastError());
        SA_CUDA_TRY(cudaMemcpy(lcp.data(), d_lcp.p, n * 4, cudaMemcpyDeviceToHost));
    }
    lcp[n] = 0;
    SA_TRY(sa_extract_sa(idx, sa.data()));
    std::vector<uint64_t> text((n + 31) / 32);
    SA_CUDA_TRY(cudaMemcpy(text.data(), idx->text, text.size() * 8, cudaMemcpyDeviceToHost));
    // ---- lcp-interval tree: bottom-up stack traversal (post-order node ids) ----
    HostTree t;
    t.lb.reserve(n / 2 + 16);
    std::vector<Frame> st;
    st.push_back(Frame{0, 0});
    auto add_child = [&](Frame &f, uint32_t c) {
        if (f.first_child == kNone) f.first_child = c; else t.sib[f.last_child] = c;
        f.last_child = c;
    };
    for (uint64_t i = 1; i <= n; ++i) {
        const uint32_t l = (i < n) ? lcp[i] : 0;
        uint32_t lb = (uint32_t)(i - 1);
        uint32_t last = kNone;
        while (l < st.back().lcp) {
            Frame f = st.back();
            st.pop_back();
            const uint32_t id = new_node(t, f.lb, (uint32_t)(i - 1), f.lcp, sa);
            fill_children(t, id, f.first_child, sa, text, n);
            lb = f.lb;
            if (l <= st.back().lcp) { add_child(st.back(), id); last = kNone; }
            else last = id;
        }
        if (l > st.back().lcp) {
            Frame f{l, lb};
            if (last != kNone) add_child(f, last);
            st.push_back(f);
        }
    }
    // the root: [0, n-1] at depth 0
    {
        Frame f = st.back();
        const uint32_t id = new_node(t, 0, (uint32_t)(n - 1), 0, sa);
        fill_children(t, id, f.first_child, sa, text, n);
    }
    sa_tree *tree = new (std::nothrow) sa_tree();
    if (!tree) { sa_set_error("host allocation failed"); return SA_ENOMEM; }
    tree->idx = idx;
    tree->nodes = t.lb.size();
    tree->root = (uint32_t)(tree->nodes - 1);
    std::vector<uint4> flat(2 * tree->nodes);
    for (uint64_t u = 0; u < tree->nodes; ++u) {
        flat[2 * u] = make_uint4(t.lb[u], t.rb[u], t.depth[u], t.pos[u]);
        flat[2 * u + 1] = make_uint4(t.child[4 * u], t.child[4 * u + 1], t.child[4 * u + 2], t.child[4 * u + 3]);
    }
    cudaError_t e = cudaMalloc(&tree->node, flat.size() * sizeof(uint4));
    if (e == cudaSuccess) e = cudaMemcpy(tree->node, flat.data(), flat.size() * sizeof(uint4), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        cudaFree(tree->node);
        delete tree;
        sa_set_error("tree upload: %s", cudaGetErrorString(e));
        return e == cudaErrorMemoryAllocation ? SA_ENOMEM : SA_ECUDA;
    }
    tree->device_bytes = flat.size() * sizeof(uint4);
    *out = tree;
    return SA_OK;
}

extern "C" void sa_tree_destroy(sa_tree *tree) {
    if (!tree) return;
    cudaFree(tree->node);
    delete tree;
}

extern "C" sa_status sa_tree_info(const sa_tree *tree, uint64_t *nodes, uint64_t *device_bytes) {
    sa_clear_error();
    if (!tree) { sa_set_error("tree is NULL"); return SA_EINVAL; }
    if (nodes) *nodes = tree->nodes;
    if (device_bytes) *device_bytes = tree->device_bytes;
    return SA_OK;
}

namespace {

struct TreeArgs {
    const uint4 *__restrict__ node;
    uint32_t root;
    const uint64_t *__restrict__ text;
    const uint32_t *__restrict__ sa;  // SA values (stride in uint32 units)
    uint32_t sa_stride;
    uint64_t n;
    const uint64_t *__restrict__ words;
    const uint32_t *__restrict__ lens;
    uint32_t fixed_len, stride;
    uint64_t Q;
    const uint32_t *__restrict__ order;
    uint32_t *__restrict__ out;
};

// range start of a child slot (internal: its lb; leaf: its rank)
__device__ __forceinline__ uint32_t child_start(const TreeArgs &a, uint32_t ch) {
    return (ch & kLeaf) ? (ch & ~kLeaf) : ld_u32(reinterpret_cast<const uint32_t *>(a.node + 2ull * ch));
}

// word j of the read (register arrays need static indices: select by unrolled compare)
template <int QW>
__device__ __forceinline__ uint64_t read_word(const sa_search::QueryWords<QW> &P, uint32_t j) {
    if constexpr (QW == 0) {
        return P.word((int)j);
    } else {
        uint64_t w = 0;
#pragma unroll
        for (int i = 0; i < QW; ++i)
            if ((uint32_t)i == j) w = P.w[i];
        return w;
    }
}

template <int QW>
__global__ void __launch_bounds__(256) k_tree_match(const TreeArgs a) {
    using namespace sa_search;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.Q) return;
    const uint64_t q = a.order ? (uint64_t)__ldg(a.order + t) : t;
    const uint32_t m = min(a.lens ? __ldg(a.lens + q) : a.fixed_len, 32u * a.stride);
    QueryWords<QW> P;
    P.load(a.words + q * a.stride, (m + 31) >> 5, false);
    uint32_t v = a.root, lo = 0, hi = 0;
    uint4 h = ld_v4u32(a.node + 2ull * v);  // {lb, rb, depth, pos}
    for (;;) {
        const uint32_t D = h.z;  // bases of P matched so far = the node's string depth
        if (m <= D) { lo = h.x; hi = h.y + 1; break; }
        const uint4 cw = ld_v4u32(a.node + 2ull * v + 1);
        const uint32_t c = (uint32_t)((read_word<QW>(P, D >> 5) >> (62 - 2 * (D & 31))) & 3u);
        const uint32_t kids[4] = {cw.x, cw.y, cw.z, cw.w};
        const uint32_t ch = kids[c];
        if (ch == kNone) {  // no edge starts with P[D]: insertion point = first child with a larger base
            uint32_t ins = h.y + 1;
            for (uint32_t c2 = 3; c2 > c; --c2)
                if (kids[c2] != kNone) ins = child_start(a, kids[c2]);
            lo = hi = ins;
            break;
        }
        if (ch & kLeaf) {  // a leaf edge: compare the rest of P with that one suffix
            const uint32_t x = ch & ~kLeaf;
            const uint64_t s = ld_u32(a.sa + (uint64_t)x * a.sa_stride);
            int sign;
            uint32_t lcp;
            compare_text<QW>(a.text, a.n, s, P, m, D, sign, lcp);
            lo = (sign > 0) ? x + 1 : x;
            hi = (sign >= 0) ? x + 1 : x;
            break;
        }
        // an internal edge: its label is the child's first suffix between depths D and depth(child)
        const uint4 hc = ld_v4u32(a.node + 2ull * ch);
        int sign;
        uint32_t lcp;
        compare_text<QW>(a.text, a.n, hc.w, P, m, D, sign, lcp);
        if (lcp < min(m, hc.z)) {  // mismatch inside the edge
            lo = hi = (sign < 0) ? hc.x : hc.y + 1;
            break;
        }
        v = ch;
        h = hc;
    }
    reinterpret_cast<uint2 *>(a.out)[q] = make_uint2(lo, hi);
}

}  // namespace

extern "C" sa_status sa_tree_match(const sa_tree *tree, const uint64_t *q_words, const uint32_t *q_len,
                                   uint32_t fixed_len, uint32_t stride_words, uint64_t Q, const uint32_t *order,
                                   uint32_t *out_lohi, void *stream) {
    sa_clear_error();
    if (!tree) { sa_set_error("tree is NULL"); return SA_EINVAL; }
    if (Q == 0) return SA_OK;
    if (!q_words || !out_lohi || stride_words == 0) { sa_set_error("bad arguments (strided reads only)"); return SA_EINVAL; }
    if (!q_len && fixed_len > 32u * stride_words) { sa_set_error("fixed_len exceeds 32*stride_words"); return SA_EINVAL; }
    const sa_index *idx = tree->idx;
    SA_CUDA_TRY(cudaSetDevice(idx->device));
    const SaView sv = sa_view(idx);
    TreeArgs a{tree->node, tree->root, idx->text, sv.base, sv.stride, idx->n, q_words, q_len, fixed_len,
               stride_words, Q, order, out_lohi};
    const unsigned blocks = (unsigned)((Q + 255) / 256);
    cudaStream_t st = (cudaStream_t)stream;
    if (stride_words <= 1) k_tree_match<1><<<blocks, 256, 0, st>>>(a);
    else if (stride_words <= 2) k_tree_match<2><<<blocks, 256, 0, st>>>(a);
    else if (stride_words <= 4) k_tree_match<4><<<blocks, 256, 0, st>>>(a);
    else k_tree_match<0><<<blocks, 256, 0, st>>>(a);
    SA_CUDA_TRY(cudaGetLastError());
    return SA_OK;
}
