// sa_api.cu -- C ABI plumbing of libsa: errors, index lifetime, exports, measurement tool.
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <new>

#include "sa_internal.cuh"

static thread_local char g_err[512] = "";

void sa_set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}
void sa_clear_error() { g_err[0] = 0; }

extern "C" const char *sa_last_error(void) { return g_err; }
extern "C" int32_t sa_version(void) { return 100; /* 0.1.0 */ }

void sa_free_index(sa_index *idx) {
    if (!idx) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(idx->device);
    cudaDeviceSynchronize();
    cudaFree(idx->text);
    cudaFree(idx->sa);
    cudaFree(idx->rec);
    cudaFree(idx->table);
    cudaFree(idx->big_hash);
    cudaFree(idx->big_sub);
    cudaFree(idx->route_table);
    cudaFree(idx->tree);
    cudaFree(idx->tree_hash);
    cudaFree(idx->part_ranks_dev);
    for (int b = 0; b < 2; ++b) {
        cudaFree(idx->pipe_words[b]);
        cudaFree(idx->pipe_lens[b]);
        cudaFree(idx->pipe_out[b]);
        cudaFree(idx->pipe_order[b]);
        cudaFree(idx->pipe_ws[b]);
        if (idx->pipe_stream[b]) cudaStreamDestroy(idx->pipe_stream[b]);
    }
    (void)cudaGetLastError();
    cudaSetDevice(prev);
    delete idx;
}
static void free_index(sa_index *idx) { sa_free_index(idx); }

extern "C" sa_status sa_index_create(const char *ref_ascii, uint64_t n, const sa_index_opts *opts, sa_index **out) {
    sa_clear_error();
    if (!out) { sa_set_error("out is NULL"); return SA_EINVAL; }
    *out = nullptr;
    if (n == 0) { sa_set_error("empty reference (n = 0)"); return SA_EEMPTY; }
    if (!ref_ascii) { sa_set_error("ref_ascii is NULL"); return SA_EINVAL; }
    if (n > 0xFFFFFFFFull) {
        sa_set_error("reference of %llu bases exceeds 2^32-1 (uint32 suffix array)", (unsigned long long)n);
        return SA_ETOOLONG;
    }
    sa_index_opts o{-1, 0, 0, 0};
    if (opts) o = *opts;
    if ((o.flags & ~(SA_INDEX_PLAIN | SA_INDEX_REC32 | SA_INDEX_BUILD_DC3 | SA_INDEX_SUBTABLE | SA_INDEX_BUCKET_TREE)) != 0 ||
        (o.flags & (SA_INDEX_PLAIN | SA_INDEX_REC32)) == (SA_INDEX_PLAIN | SA_INDEX_REC32) || o.reserved != 0) {
        sa_set_error("unknown opts.flags bits / reserved must be 0");
        return SA_EINVAL;
    }
    if ((o.flags & SA_INDEX_BUCKET_TREE) && (!(o.flags & SA_INDEX_REC32) || (o.flags & SA_INDEX_SUBTABLE))) {
        sa_set_error("SA_INDEX_BUCKET_TREE needs SA_INDEX_REC32 and excludes SA_INDEX_SUBTABLE");
        return SA_EINVAL;
    }
    if (o.kmer_k > 16) { sa_set_error("kmer_k %u out of range 1..16", o.kmer_k); return SA_EINVAL; }
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
        (void)cudaGetLastError();
        sa_set_error("no CUDA device available (%s)", e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
        return SA_ECUDA;
    }
    int dev = o.device;
    if (dev < 0) SA_CUDA_TRY(cudaGetDevice(&dev));
    if (dev >= ndev) { sa_set_error("device %d out of range (%d devices)", dev, ndev); return SA_EINVAL; }
    int prev = 0;
    SA_CUDA_TRY(cudaGetDevice(&prev));
    SA_CUDA_TRY(cudaSetDevice(dev));

    sa_index *idx = new (std::nothrow) sa_index();
    if (!idx) { sa_set_error("host allocation failed"); cudaSetDevice(prev); return SA_ENOMEM; }
    idx->device = dev;
    idx->n = n;
    idx->layout = (o.flags & SA_INDEX_PLAIN) ? 0 : (o.flags & SA_INDEX_REC32) ? 2 : 1;
    idx->build_dc3 = (o.flags & SA_INDEX_BUILD_DC3) != 0;
    idx->subtables = (o.flags & SA_INDEX_SUBTABLE) != 0;
    idx->bucket_tree = (o.flags & SA_INDEX_BUCKET_TREE) != 0;
    uint32_t k = o.kmer_k;
    if (k == 0) {  // auto: floor(log4 n) + 1 (mean bracket < 1 suffix), at most 16 (a 16 GiB table)
        k = 1;
        while (k < 16 && (1ull << (2 * k)) <= n) ++k;
    }
    idx->k = k;
    cudaStream_t st = nullptr;
    sa_status s = SA_OK;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
        (void)cudaGetLastError();
        sa_set_error("stream creation failed");
        s = SA_ECUDA;
    }
    if (s == SA_OK) s = sa_build_index(idx, ref_ascii, st);
    if (st) {
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
    }
    if (s != SA_OK) {
        free_index(idx);
        cudaSetDevice(prev);
        return s;
    }
    cudaSetDevice(prev);
    *out = idx;
    return SA_OK;
}

extern "C" void sa_index_destroy(sa_index *idx) { free_index(idx); }

extern "C" sa_status sa_dc3_trace(const char *ref_ascii, uint64_t n, uint32_t *sample_rank, uint32_t *nonsample) {
    sa_clear_error();
    if (!ref_ascii || n == 0) { sa_set_error("empty or NULL reference"); return SA_EINVAL; }
    if (n > 0xFFFFFFFFull) { sa_set_error("reference too long"); return SA_ETOOLONG; }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        (void)cudaGetLastError();
        sa_set_error("no CUDA device available");
        return SA_ECUDA;
    }
    sa_index *idx = new (std::nothrow) sa_index();
    if (!idx) return SA_ENOMEM;
    SA_CUDA_TRY(cudaGetDevice(&idx->device));
    idx->n = n;
    cudaStream_t st = nullptr;
    sa_status s = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) == cudaSuccess ? SA_OK : SA_ECUDA;
    if (s == SA_OK) s = sa_pack_text(idx, ref_ascii, st);
    if (s == SA_OK && cudaMalloc(&idx->sa, n * sizeof(uint32_t)) != cudaSuccess) { (void)cudaGetLastError(); s = SA_ENOMEM; }
    if (s == SA_OK) s = sa_build_sa_dc3(idx, st, sample_rank, nonsample);
    if (st) { cudaStreamSynchronize(st); cudaStreamDestroy(st); }
    free_index(idx);
    return s;
}

extern "C" sa_status sa_index_info(const sa_index *idx, uint64_t *n, uint32_t *kmer_k, uint64_t *device_bytes,
                                   int32_t *device) {
    sa_clear_error();
    if (!idx) { sa_set_error("index is NULL"); return SA_EINVAL; }
    if (n) *n = idx->n;
    if (kmer_k) *kmer_k = idx->k;
    if (device_bytes) *device_bytes = idx->device_bytes;
    if (device) *device = idx->device;
    return SA_OK;
}

static sa_status export_copy(const sa_index *idx, void *dst, const void *src, size_t bytes) {
    if (!idx || !dst) { sa_set_error("NULL argument"); return SA_EINVAL; }
    SA_CUDA_TRY(cudaSetDevice(idx->device));
    SA_CUDA_TRY(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
    return SA_OK;
}

extern "C" sa_status sa_index_export_sa(const sa_index *idx, uint32_t *host_out) {
    sa_clear_error();
    if (!idx || !host_out) { sa_set_error("NULL argument"); return SA_EINVAL; }
    SA_CUDA_TRY(cudaSetDevice(idx->device));
    return sa_extract_sa(idx, host_out);  // (a partition: its slice SA[rank_lo .. rank_hi))
}

extern "C" sa_status sa_index_export_table(const sa_index *idx, uint32_t *host_out) {
    sa_clear_error();
    // a partition: its slice T[x_lo .. x_hi] (sa_index_part_info)
    const uint64_t entries = !idx ? 0 : idx->nparts > 1 ? idx->table_entries : (1ull << (2 * idx->k)) + 1;
    return export_copy(idx, host_out, idx ? idx->table : nullptr, entries * sizeof(uint32_t));
}

extern "C" sa_status sa_index_export_text(const sa_index *idx, uint64_t *host_out) {
    sa_clear_error();
    return export_copy(idx, host_out, idx ? idx->text : nullptr, idx ? ((idx->n + 31) / 32) * sizeof(uint64_t) : 0);
}

// ---- measurement tool: random-access gather rate ---------------------------------------------
__device__ __forceinline__ uint64_t hash64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Each thread issues `loads` loads in groups of 8 independent addresses (slots is a power of two,
// so the address is one hash + mask); dependent = 1 chains every address on the previous value.
template <int BYTES>
__global__ void k_gather(const uint8_t *__restrict__ buf, uint64_t slot_mask, uint32_t loads, int dependent,
                         uint64_t *__restrict__ sink) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t acc = 0;
    uint64_t h = hash64(tid * 0x9E3779B97F4A7C15ull + 0x1234567ull);
    for (uint32_t i = 0; i < loads; i += 8) {
        uint64_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint64_t slot = (dependent ? hash64(h + acc + u) : hash64(h + i + u)) & slot_mask;
            const uint8_t *p = buf + slot * BYTES;
            if constexpr (BYTES == 32) {
                const ulonglong4 x = *reinterpret_cast<const ulonglong4 *>(p);  // 256-bit load (sm_100)
                v[u] = x.x ^ x.y ^ x.z ^ x.w;
            } else if constexpr (BYTES == 16) {
                const uint4 x = __ldg(reinterpret_cast<const uint4 *>(p));
                v[u] = (uint64_t)x.x ^ x.y ^ x.z ^ x.w;
            } else if constexpr (BYTES == 8) {
                v[u] = __ldg(reinterpret_cast<const unsigned long long *>(p));
            } else {
                v[u] = __ldg(reinterpret_cast<const unsigned int *>(p));
            }
            if (dependent) acc += v[u];
        }
        if (!dependent) {
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += v[u];
        }
    }
    if (acc == 0x5eed) sink[0] = acc;  // keeps the loads alive
}

// modes 10..13: independent random loads with an explicit PTX cache operator (measurement of the
// DRAM bytes one random access costs): 10 ld.global.nc, 11 ld.global.cg, 12 ld.global.cv,
// 13 ld.global.nc.L1::no_allocate; BYTES = 8 or 32.
template <int BYTES, int OP>
__device__ __forceinline__ uint64_t ld_op(const uint8_t *p) {
    uint64_t a = 0, b = 0, c = 0, d = 0;
    if constexpr (BYTES == 32) {
        if constexpr (OP == 0) asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
        if constexpr (OP == 1) asm volatile("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
        if constexpr (OP == 2) asm volatile("ld.global.cv.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
        if constexpr (OP == 3) asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
        return a ^ b ^ c ^ d;
    } else {
        if constexpr (OP == 0) asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(a) : "l"(p));
        if constexpr (OP == 1) asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(a) : "l"(p));
        if constexpr (OP == 2) asm volatile("ld.global.cv.u64 %0, [%1];" : "=l"(a) : "l"(p));
        if constexpr (OP == 3) asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(a) : "l"(p));
        return a;
    }
}

template <int BYTES, int OP>
__global__ void k_gather_op(const uint8_t *__restrict__ buf, uint64_t slot_mask, uint32_t loads,
                            uint64_t *__restrict__ sink) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t acc = 0;
    const uint64_t h = hash64(tid * 0x9E3779B97F4A7C15ull + 0x1234567ull);
    for (uint32_t i = 0; i < loads; i += 8) {
        uint64_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = ld_op<BYTES, OP>(buf + (hash64(h + i + u) & slot_mask) * BYTES);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u];
    }
    if (acc == 0x5eed) sink[0] = acc;
}

// modes 20..22: the same 32-byte random loads through the asynchronous copy paths, to see whether a
// path that is not an LSU load moves fewer than the 4 DRAM sectors an LSU load costs:
// 20 cp.async.bulk (TMA bulk copy, 32 B into shared memory, mbarrier completion), 21 cp.async.cg
// (LDGSTS, two 16-byte copies), 22 ld.global.nc.L2::64B (prefetch-size hint).
template <int OP>
__global__ void __launch_bounds__(128) k_gather_async(const uint8_t *__restrict__ buf, uint64_t slot_mask,
                                                      uint32_t loads, uint64_t *__restrict__ sink) {
    __shared__ __align__(128) ulonglong4 stage[128 * 8];
    __shared__ __align__(8) uint64_t bar[4];
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[warp]);
    if constexpr (OP == 20) {
        if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        __syncwarp();
    }
    ulonglong4 *mine = stage + threadIdx.x * 8;
    uint64_t acc = 0;
    uint32_t phase = 0;
    const uint64_t h = hash64(tid * 0x9E3779B97F4A7C15ull + 0x1234567ull);
    for (uint32_t i = 0; i < loads; i += 8) {
        if constexpr (OP == 22) {
            uint64_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint8_t *p = buf + (hash64(h + i + u) & slot_mask) * 32;
                uint64_t a, c, d, e;
                asm volatile("ld.global.nc.L2::64B.v4.u64 {%0,%1,%2,%3}, [%4];"
                             : "=l"(a), "=l"(c), "=l"(d), "=l"(e) : "l"(p));
                v[u] = a ^ c ^ d ^ e;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += v[u];
            continue;
        }
        if constexpr (OP == 20) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(8 * 32) : "memory");
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint8_t *p = buf + (hash64(h + i + u) & slot_mask) * 32;
                const uint32_t dst = (uint32_t)__cvta_generic_to_shared(mine + u);
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 32, [%2];"
                             ::"r"(dst), "l"(p), "r"(b) : "memory");
            }
            uint32_t done = 0;
            while (!done) {
                asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                             : "=r"(done) : "r"(b), "r"(phase) : "memory");
            }
            phase ^= 1;
        } else {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint8_t *p = buf + (hash64(h + i + u) & slot_mask) * 32;
                const uint32_t dst = (uint32_t)__cvta_generic_to_shared(mine + u);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(p) : "memory");
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16), "l"(p + 16) : "memory");
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += mine[u].x ^ mine[u].w;
        __syncwarp();
    }
    if (acc == 0x5eed) sink[0] = acc + lane;
}

// mode 2: random stores of BYTES (partial-sector stores below 32 B exercise the L2 / ECC
// read-modify-write path of a scattered result write)
template <int BYTES>
__global__ void k_scatter(uint8_t *__restrict__ buf, uint64_t slot_mask, uint32_t stores) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t h = hash64(tid * 0x9E3779B97F4A7C15ull + 0x7654321ull);
    for (uint32_t i = 0; i < stores; ++i) {
        const uint64_t slot = hash64(h + i) & slot_mask;
        uint8_t *p = buf + slot * BYTES;
        if constexpr (BYTES == 32) {
            *reinterpret_cast<ulonglong4 *>(p) = make_ulonglong4(h, i, tid, slot);
        } else if constexpr (BYTES == 16) {
            *reinterpret_cast<uint4 *>(p) = make_uint4((uint32_t)h, i, (uint32_t)tid, (uint32_t)slot);
        } else if constexpr (BYTES == 8) {
            *reinterpret_cast<unsigned long long *>(p) = h + i;
        } else {
            *reinterpret_cast<unsigned int *>(p) = (uint32_t)(h + i);
        }
    }
}

extern "C" sa_status sa_tool_random_gather(int32_t device, uint64_t buffer_bytes, uint32_t access_bytes,
                                           uint64_t n_threads, uint32_t loads, int32_t dependent, float *ms) {
    sa_clear_error();
    if (!ms || buffer_bytes < 4096 || n_threads == 0 || loads == 0 ||
        !(access_bytes == 4 || access_bytes == 8 || access_bytes == 16 || access_bytes == 32)) {
        sa_set_error("bad argument");
        return SA_EINVAL;
    }
    SA_CUDA_TRY(cudaSetDevice(device));
    // measurement knob of this tool only: SA_L2_FETCH_BYTES=32|64|128 -> cudaLimitMaxL2FetchGranularity
    if (const char *g = getenv("SA_L2_FETCH_BYTES")) {
        const int b = atoi(g);
        if (b == 32 || b == 64 || b == 128) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)b);
        (void)cudaGetLastError();
    }
    uint8_t *buf = nullptr;
    uint64_t *sink = nullptr;
    SA_CUDA_TRY(cudaMalloc(&buf, buffer_bytes));
    if (cudaMalloc(&sink, 8) != cudaSuccess) { cudaFree(buf); SA_CUDA_TRY(cudaGetLastError()); }
    cudaMemset(buf, 0x5A, buffer_bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    uint64_t slots = 1;
    while (slots * 2 * access_bytes <= buffer_bytes) slots *= 2;  // power of two: address = hash & mask
    const unsigned threads = 256;
    const unsigned blocks = (unsigned)((n_threads + threads - 1) / threads);
    auto launch = [&]() {
        if (dependent >= 10 && dependent <= 13 && (access_bytes == 32 || access_bytes == 8)) {
            const int op = dependent - 10;
#define SA_GOP(B, O) k_gather_op<B, O><<<blocks, threads>>>(buf, slots - 1, loads, sink)
            if (access_bytes == 32) {
                if (op == 0) SA_GOP(32, 0); else if (op == 1) SA_GOP(32, 1); else if (op == 2) SA_GOP(32, 2); else SA_GOP(32, 3);
            } else {
                if (op == 0) SA_GOP(8, 0); else if (op == 1) SA_GOP(8, 1); else if (op == 2) SA_GOP(8, 2); else SA_GOP(8, 3);
            }
#undef SA_GOP
            return;
        }
        if (dependent >= 20 && dependent <= 22 && access_bytes == 32) {
            const unsigned b2 = blocks * 2;  // 128-thread blocks (64 KB of staging would not fit otherwise)
            if (dependent == 20) k_gather_async<20><<<b2, 128>>>(buf, slots - 1, loads, sink);
            else if (dependent == 21) k_gather_async<21><<<b2, 128>>>(buf, slots - 1, loads, sink);
            else k_gather_async<22><<<b2, 128>>>(buf, slots - 1, loads, sink);
            return;
        }
        if (dependent == 2) {
            switch (access_bytes) {
            case 32: k_scatter<32><<<blocks, threads>>>(buf, slots - 1, loads); break;
            case 16: k_scatter<16><<<blocks, threads>>>(buf, slots - 1, loads); break;
            case 8: k_scatter<8><<<blocks, threads>>>(buf, slots - 1, loads); break;
            default: k_scatter<4><<<blocks, threads>>>(buf, slots - 1, loads); break;
            }
            return;
        }
        switch (access_bytes) {
        case 32: k_gather<32><<<blocks, threads>>>(buf, slots - 1, loads, dependent, sink); break;
        case 16: k_gather<16><<<blocks, threads>>>(buf, slots - 1, loads, dependent, sink); break;
        case 8: k_gather<8><<<blocks, threads>>>(buf, slots - 1, loads, dependent, sink); break;
        default: k_gather<4><<<blocks, threads>>>(buf, slots - 1, loads, dependent, sink); break;
        }
    };
    launch();  // warm-up
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float t = 0;
    cudaEventElapsedTime(&t, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(buf);
    cudaFree(sink);
    SA_CUDA_TRY(e);
    SA_CUDA_TRY(cudaGetLastError());
    *ms = t;
    return SA_OK;
}
