// Embedding backward (backward_embedding, proj/src/executor.cpp:1199-1219):
// gtable[row] += sum of g over positions with llround(id) mod V == row, rows
// outside this rank's vocab slice skipped. Deterministic (no float atomics)
// and parallel even when the ids are heavily repeated (the reference's
// synthetic ids hit ~9 rows):
//   1. keys (row << 32 | position) are sorted — by one block in shared memory, or for
//      N >= 4096 as 1024-key runs (one block each) merged by rank — and one block
//      cuts the sorted order into "pieces": maximal runs of one row inside an
//      aligned 64-position chunk (piece starts, rows, segment-head flags);
//   2. one block per (piece, 256 dims) sums its <= 64 gradient rows in order;
//   3. the first piece of each row-segment adds its segment's piece sums, in
//      piece order, into the table gradient.
#include "common.cuh"

namespace sbk {

namespace {
constexpr int kChunk = 64;
constexpr int kSortMax = 16384;  // keys sorted in shared memory (128 KB)

__device__ __forceinline__ i64 e_row(double raw, i64 V) {
    i64 i = (i64)llround(raw) % V;
    return i < 0 ? i + V : i;
}

i64 pow2_ge(i64 n) {
    i64 p = 1;
    while (p < n) p <<= 1;
    return p;
}

struct Layout {
    unsigned long long* keys;    // N (global fallback sort; sorted 1024-key runs)
    unsigned long long* sorted;  // N (merged runs)
    int* piece_start;          // npieces + 1
    int* piece_row;
    int* piece_head;
    int* npieces;
    int* perm;                 // sorted positions (n)
    float* piece_sum;          // npieces_max * dim
};

Layout carve(void* ws, i64 n, i64 dim) {
    char* p = (char*)ws;
    Layout L;
    i64 N = pow2_ge(std::max<i64>(n, 1));
    L.keys = (unsigned long long*)p;
    p += N * 8;
    L.sorted = (unsigned long long*)p;
    p += N * 8;
    i64 pmax = n / kChunk + n + 2;
    L.piece_start = (int*)p;
    p += (pmax + 1) * 4;
    L.piece_row = (int*)p;
    p += pmax * 4;
    L.piece_head = (int*)p;
    p += pmax * 4;
    L.npieces = (int*)p;
    p += 16;
    L.perm = (int*)p;
    p += n * 4;
    p = (char*)(((uintptr_t)p + 255) & ~(uintptr_t)255);
    L.piece_sum = (float*)p;
    return L;
}

// key of position i: (row << 32 | i); positions outside this rank's rows (and the
// padding up to N) get row 0xFFFFFFFF: unique keys that sort last
__device__ __forceinline__ unsigned long long e_key(const double* ids, i64 i, i64 n, i64 V, i64 row0, i64 local) {
    unsigned long long k = (0xFFFFFFFFull << 32) | (unsigned long long)i;
    if (i < n) {
        i64 r = e_row(ids[i], V) - row0;
        if (r >= 0 && r < local) k = ((unsigned long long)r << 32) | (unsigned long long)i;
    }
    return k;
}
__device__ __forceinline__ bool e_invalid(unsigned long long k) { return (k >> 32) == 0xFFFFFFFFull; }

// large N: every block sorts one 1024-key run in shared memory ...
__global__ void __launch_bounds__(1024) k_emb_runs(const double* ids, i64 n, i64 V, i64 row0, i64 local, Layout L) {
    __shared__ unsigned long long k[1024];
    const int t = threadIdx.x;
    const i64 base = (i64)blockIdx.x * 1024;
    k[t] = e_key(ids, base + t, n, V, row0, local);
    __syncthreads();
    for (int size = 2; size <= 1024; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const int j = t ^ stride;
            if (j > t) {
                const bool up = (t & size) == 0;
                const unsigned long long a = k[t], b = k[j];
                if ((a > b) == up) {
                    k[t] = b;
                    k[j] = a;
                }
            }
            __syncthreads();
        }
    L.keys[base + t] = k[t];
}
// ... then each key's final position is its position in its run plus, per other run,
// the number of (unique) keys below it (binary search)
__global__ void k_emb_merge(i64 N, Layout L) {
    const i64 g = blockIdx.x * (i64)blockDim.x + threadIdx.x;
    if (g >= N) return;
    const unsigned long long key = L.keys[g];
    const i64 run = g / 1024, nruns = N / 1024;
    i64 rank = g % 1024;
    for (i64 r = 0; r < nruns; ++r) {
        if (r == run) continue;
        const unsigned long long* a = L.keys + r * 1024;
        int lo = 0, hi = 1024;  // first element >= key
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (a[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        rank += lo;
    }
    L.sorted[rank] = key;
}

__global__ void __launch_bounds__(1024) k_emb_pieces(const double* ids, i64 n, i64 N, i64 V, i64 row0, i64 local,
                                                     Layout L, int use_smem) {
    extern __shared__ unsigned long long skeys[];
    // use_smem 2: keys already sorted in L.sorted (k_emb_runs + k_emb_merge)
    unsigned long long* keys = use_smem == 2 ? L.sorted : use_smem ? skeys : L.keys;
    __shared__ int warp_tot[32];
    if (use_smem != 2) {
    for (i64 i = threadIdx.x; i < N; i += blockDim.x) keys[i] = e_key(ids, i, n, V, row0, local);
    __syncthreads();
    for (i64 size = 2; size <= N; size <<= 1)
        for (i64 stride = size >> 1; stride > 0; stride >>= 1) {
            for (i64 i = threadIdx.x; i < N; i += blockDim.x) {
                i64 j = i ^ stride;
                if (j > i) {
                    bool up = (i & size) == 0;
                    unsigned long long a = keys[i], b = keys[j];
                    if ((a > b) == up) {
                        keys[i] = b;
                        keys[j] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    // piece flags over the valid prefix, block-wide exclusive scan (ordered)
    const int per = (int)((n + blockDim.x - 1) / blockDim.x);
    const i64 lo = (i64)threadIdx.x * per, hi = min(lo + per, n);
    __shared__ int s_nvalid;
    if (threadIdx.x == 0) s_nvalid = 0;
    __syncthreads();
    int cnt = 0, nv = 0;  // pieces starting in / valid keys of [lo, hi) (valid keys are a prefix)
    for (i64 m = lo; m < hi; ++m) {
        unsigned long long k = keys[m];
        if (e_invalid(k)) break;
        bool flag = (m % kChunk == 0) || (keys[m - 1] >> 32) != (k >> 32);
        cnt += flag;
        ++nv;
    }
    if (nv) atomicAdd(&s_nvalid, nv);  // integer count: order-independent
    // scan of cnt across the block
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = cnt;
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
        int v = lane < (int)(blockDim.x / 32) ? warp_tot[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        warp_tot[lane] = v;
    }
    __syncthreads();
    int base = x - cnt + (w > 0 ? warp_tot[w - 1] : 0);
    int total = warp_tot[(blockDim.x / 32) - 1];
    for (i64 m = lo; m < hi; ++m) {
        unsigned long long k = keys[m];
        if (e_invalid(k)) break;
        L.perm[m] = (int)(k & 0xffffffffull);
        bool rowchg = m == 0 || (keys[m - 1] >> 32) != (k >> 32);
        if ((m % kChunk == 0) || rowchg) {
            L.piece_start[base] = (int)m;
            L.piece_row[base] = (int)(k >> 32);
            L.piece_head[base] = rowchg;
            ++base;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        L.piece_start[total] = s_nvalid;  // end of the valid region closes the last piece
        *L.npieces = total;
    }
}

template <class T>
__global__ void k_emb_piece_sum(Layout L, const T* g, i64 dim) {
    int p = blockIdx.x;
    if (p >= *L.npieces) return;
    i64 d = blockIdx.y * (i64)blockDim.x + threadIdx.x;
    if (d >= dim) return;
    int s = L.piece_start[p], e = L.piece_start[p + 1];
    float acc = 0.f;
    for (int m = s; m < e; ++m) acc += to_f(g[(i64)L.perm[m] * dim + d]);
    L.piece_sum[(i64)p * dim + d] = acc;
}

__global__ void k_emb_combine(Layout L, i64 dim, float* gt) {
    int p = blockIdx.x;
    int np = *L.npieces;
    if (p >= np || !L.piece_head[p]) return;
    i64 d = blockIdx.y * (i64)blockDim.x + threadIdx.x;
    if (d >= dim) return;
    int row = L.piece_row[p];
    int q1 = p + 1;  // end of this row's segment
    while (q1 < np && L.piece_row[q1] == row && !L.piece_head[q1]) ++q1;
    float acc = 0.f;
    int q = p;
    for (; q + 8 <= q1; q += 8) {  // 8 loads in flight, summed in piece order
        float a[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] = L.piece_sum[(i64)(q + u) * dim + d];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += a[u];
    }
    for (; q < q1; ++q) acc += L.piece_sum[(i64)q * dim + d];
    gt[(i64)row * dim + d] += acc;
}
}  // namespace

size_t embedding_bwd_workspace(i64 n, i64 dim) {
    i64 N = pow2_ge(std::max<i64>(n, 1));
    i64 pmax = n / kChunk + n + 2;
    return (size_t)(2 * N * 8 + (pmax + 1) * 4 + 2 * pmax * 4 + 16 + n * 4 + 256 + pmax * dim * 4);
}

void embedding_bwd(const double* ids, i64 n, const void* g, DT tg, i64 dim, i64 V, i64 row0, i64 local, float* gt,
                   void* ws, cudaStream_t s) {
    if (n == 0) return;
    Layout L = carve(ws, n, dim);
    i64 N = pow2_ge(n);
    int use_smem = N <= kSortMax;
    size_t smem = use_smem ? (size_t)N * 8 : 0;
    if (N >= 4096) {  // parallel: sorted 1024-key runs, merged by rank
        k_emb_runs<<<(unsigned)(N / 1024), 1024, 0, s>>>(ids, n, V, row0, local, L);
        k_emb_merge<<<(unsigned)(N / 256), 256, 0, s>>>(N, L);
        use_smem = 2;
        smem = 0;
    }
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_emb_pieces, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_emb_pieces<<<1, 1024, smem, s>>>(ids, n, N, V, row0, local, L, use_smem);
    i64 pmax = n / kChunk + std::min(n, local) + 2;
    dim3 grid((unsigned)pmax, (unsigned)((dim + 255) / 256));
    dispatch(tg, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        k_emb_piece_sum<T><<<grid, 256, 0, s>>>(L, (const T*)g, dim);
    });
    k_emb_combine<<<grid, 256, 0, s>>>(L, dim, gt);
    SBK_CHECK_LAUNCH();
}

}  // namespace sbk
