// kernels_scan.cu -- device-wide exclusive prefix sums used by the table index (int32, in place)
// and by the tile bins (uint32 counts -> uint64 offsets).  Three phases: per-chunk reduction,
// one-CTA scan of the chunk sums, per-chunk scan with the chunk offset.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>

#include "internal.h"

namespace wasabi {
namespace {

constexpr int kThreads = 1024;
constexpr int kItems = 4;
constexpr int kChunk = kThreads * kItems;

template <typename T>
__device__ T block_excl_scan(T v, T *sh, T *total) {
    // warp inclusive scan
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[wid] = x;
    __syncthreads();
    if (wid == 0) {
        T w = (lane < (int)(blockDim.x >> 5)) ? sh[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        sh[lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    const T warp_off = wid ? sh[wid - 1] : T(0);
    if (total) *total = sh[(blockDim.x >> 5) - 1];
    __syncthreads();
    return warp_off + x - v;
}

template <typename Tin, typename Tacc>
__global__ void __launch_bounds__(kThreads) reduce_chunks(const Tin *in, int64_t n, Tacc *sums) {
    __shared__ Tacc sh[32];
    const int64_t base = (int64_t)blockIdx.x * kChunk + (int64_t)threadIdx.x * kItems;
    Tacc s = 0;
#pragma unroll
    for (int i = 0; i < kItems; i++)
        if (base + i < n) s += (Tacc)in[base + i];
    Tacc tot;
    block_excl_scan<Tacc>(s, sh, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

template <typename Tacc>
__global__ void __launch_bounds__(kThreads) scan_sums(Tacc *sums, int64_t m) {
    __shared__ Tacc sh[32];
    Tacc carry = 0;
    for (int64_t b0 = 0; b0 < m; b0 += kThreads) {
        const int64_t i = b0 + threadIdx.x;
        const Tacc v = i < m ? sums[i] : Tacc(0);
        Tacc tot;
        const Tacc ex = block_excl_scan<Tacc>(v, sh, &tot);
        if (i < m) sums[i] = carry + ex;
        carry += tot;
        __syncthreads();
    }
}

template <typename Tin, typename Tout>
__global__ void __launch_bounds__(kThreads) scan_chunks(const Tin *in, Tout *out, int64_t n, const Tout *sums) {
    __shared__ Tout sh[32];
    const int64_t base = (int64_t)blockIdx.x * kChunk + (int64_t)threadIdx.x * kItems;
    Tout v[kItems];
    Tout s = 0;
#pragma unroll
    for (int i = 0; i < kItems; i++) {
        v[i] = (base + i < n) ? (Tout)in[base + i] : Tout(0);
        s += v[i];
    }
    Tout ex = block_excl_scan<Tout>(s, sh, nullptr) + sums[blockIdx.x];
#pragma unroll
    for (int i = 0; i < kItems; i++) {
        if (base + i < n) out[base + i] = ex;
        ex += v[i];
    }
}

struct Blob {
    uint32_t n, pad;
    unsigned char data[3968];
};

__global__ void write_blob_kernel(unsigned char *dst, Blob b) {
    for (uint32_t i = threadIdx.x; i < b.n; i += blockDim.x) dst[i] = b.data[i];
}

}  // namespace

// Asynchronous, graph-capturable host->device copy of small descriptors through kernel parameters
// (no pageable-memcpy stream synchronisation).
cudaError_t launch_write_blob(void *dst, const void *src, size_t bytes, cudaStream_t s) {
    // large descriptor arrays (thousands of offset-class tables): one stream-ordered copy from the
    // (pageable) host array instead of hundreds of parameter-blob launches; the call returns once
    // the source has been staged, so the caller may free it
    // -- but not while the stream is being captured into a CUDA graph: a captured memcpy node would
    // read the (by then freed) host array at every replay, so under capture the bytes always travel
    // by value in kernel parameters
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaError_t e = cudaStreamIsCapturing(s, &cap);
    if (e != cudaSuccess) return e;
    if (bytes > 16384 && cap == cudaStreamCaptureStatusNone)
        return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
    const unsigned char *p = static_cast<const unsigned char *>(src);
    unsigned char *d = static_cast<unsigned char *>(dst);
    for (size_t off = 0; off < bytes; off += sizeof(Blob::data)) {
        Blob b;
        b.n = (uint32_t)std::min(sizeof(Blob::data), bytes - off);
        b.pad = 0;
        for (uint32_t i = 0; i < b.n; i++) b.data[i] = p[off + i];
        count_launches(1);
        write_blob_kernel<<<1, 256, 0, s>>>(d + off, b);
    }
    return cudaGetLastError();
}

size_t scan_scratch_bytes(int64_t n) {
    const int64_t m = (n + kChunk - 1) / kChunk;
    return (size_t)((m + 1) * 8 + 256);
}

// In-place exclusive scan of int32 counts (the table pointer index).
cudaError_t launch_scan_i32(int32_t *data, int64_t n, void *scratch, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int64_t m = (n + kChunk - 1) / kChunk;
    int32_t *sums = reinterpret_cast<int32_t *>(scratch);
    count_launches(1);
    reduce_chunks<int32_t, int32_t><<<(unsigned)m, kThreads, 0, s>>>(data, n, sums);
    count_launches(1);
    scan_sums<int32_t><<<1, kThreads, 0, s>>>(sums, m);
    count_launches(1);
    scan_chunks<int32_t, int32_t><<<(unsigned)m, kThreads, 0, s>>>(data, data, n, sums);
    return cudaGetLastError();
}

// Exclusive scan of uint32 tile counts into uint64 offsets (out has n + 1 entries: the last
// entry, whose input count is 0 by construction, receives the total).
cudaError_t launch_scan_u32_to_u64(const uint32_t *in, unsigned long long *out, int64_t n, void *scratch,
                                   cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int64_t m = (n + kChunk - 1) / kChunk;
    unsigned long long *sums = reinterpret_cast<unsigned long long *>(scratch);
    count_launches(1);
    reduce_chunks<uint32_t, unsigned long long><<<(unsigned)m, kThreads, 0, s>>>(in, n, sums);
    count_launches(1);
    scan_sums<unsigned long long><<<1, kThreads, 0, s>>>(sums, m);
    count_launches(1);
    scan_chunks<uint32_t, unsigned long long><<<(unsigned)m, kThreads, 0, s>>>(in, out, n, sums);
    return cudaGetLastError();
}

}  // namespace wasabi
