// LDG/STG copy-engine variants on the 7B-4k migration layout (DESIGN.md §4 K1,
// "ldg" engine at 0.89 of the copy roofline).  Standalone probe: 64 planes
// (32 layers x K/V) x 256 blocks x 128 KiB pieces, block ids through an index
// array like the real kernel, 32 KiB tiles, grid = SMs x occupancy, grid-stride.
// Variants: threads per CTA x 16-byte vectors per thread per tile, and a
// two-tile software pipeline (loads of tile t+1 issued before stores of t).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_probe_ldg_copy tools/probe_ldg_copy.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kTile = 32 * 1024;
constexpr int kPiece = 128 * 1024;
constexpr int kTpp = kPiece / kTile;
constexpr int kBlocks = 256, kPlanes = 64, kPoolBlocks = 1024;

__device__ __forceinline__ int4 ldg(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void stg(int4* p, const int4& v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w) : "memory");
}

struct Args { const uint8_t* src; uint8_t* dst; const int* sb; const int* db; int64_t plane; int tiles; };

__device__ __forceinline__ void tile_ptrs(const Args& a, int t, const int4*& s, int4*& d) {
  const int per_plane = kBlocks * kTpp;
  const int plane = t / per_plane, r = t - plane * per_plane, bi = r / kTpp, ti = r - bi * kTpp;
  s = reinterpret_cast<const int4*>(a.src + plane * a.plane + (int64_t)__ldg(a.sb + bi) * kPiece + ti * kTile);
  d = reinterpret_cast<int4*>(a.dst + plane * a.plane + (int64_t)__ldg(a.db + bi) * kPiece + ti * kTile);
}

template <int kThreads, int kMinBlocks>
__global__ void __launch_bounds__(kThreads, kMinBlocks) copy_plain(const __grid_constant__ Args a) {
  constexpr int kVec = kTile / 16 / kThreads;
  for (int t = blockIdx.x; t < a.tiles; t += gridDim.x) {
    const int4* s; int4* d;
    tile_ptrs(a, t, s, d);
    int4 v[kVec];
#pragma unroll
    for (int k = 0; k < kVec; ++k) v[k] = ldg(s + threadIdx.x + k * kThreads);
#pragma unroll
    for (int k = 0; k < kVec; ++k) stg(d + threadIdx.x + k * kThreads, v[k]);
  }
}

// next tile's addresses resolved (and its loads issued) before this tile's stores
template <int kThreads>
__global__ void __launch_bounds__(kThreads) copy_pipe(const __grid_constant__ Args a) {
  constexpr int kVec = kTile / 16 / kThreads;
  int t = blockIdx.x;
  if (t >= a.tiles) return;
  const int4* s; int4* d;
  tile_ptrs(a, t, s, d);
  int4 v[kVec];
#pragma unroll
  for (int k = 0; k < kVec; ++k) v[k] = ldg(s + threadIdx.x + k * kThreads);
  for (;;) {
    const int tn = t + gridDim.x;
    const int4* sn = nullptr; int4* dn = nullptr;
    int4 w[kVec];
    if (tn < a.tiles) {
      tile_ptrs(a, tn, sn, dn);
#pragma unroll
      for (int k = 0; k < kVec; ++k) w[k] = ldg(sn + threadIdx.x + k * kThreads);
    }
#pragma unroll
    for (int k = 0; k < kVec; ++k) stg(d + threadIdx.x + k * kThreads, v[k]);
    if (tn >= a.tiles) break;
#pragma unroll
    for (int k = 0; k < kVec; ++k) v[k] = w[k];
    t = tn; s = sn; d = dn;
  }
}

template <class K>
void bench(const char* name, K kernel, int threads, const Args& a, cudaStream_t st, uint8_t* flush, size_t fbytes) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, 0);
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * occ;
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, kernel);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) kernel<<<grid, threads, 0, st>>>(a);
  float total = 0; const int iters = 20;
  for (int i = 0; i < iters; ++i) {
    cudaMemsetAsync(flush, i, fbytes, st);   // L2 flush between launches
    cudaEventRecord(e0, st);
    kernel<<<grid, threads, 0, st>>>(a);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); total += ms;
  }
  const double bytes = 2.0 * kPlanes * kBlocks * (double)kPiece;
  const double us = total / iters * 1e3;
  printf("%-28s regs %3d occ %d grid %4d: %8.1f us  %7.1f GB/s r+w (payload %.1f)\n", name, fa.numRegs, occ, grid,
         us, bytes / us / 1e3, bytes / 2 / us / 1e3);
}

int main() {
  const int64_t plane = (int64_t)kPoolBlocks * kPiece;
  const size_t pool = (size_t)plane * kPlanes;   // 8 GiB
  uint8_t* p; cudaMalloc(&p, pool);
  uint8_t* flush; const size_t fbytes = 256u << 20; cudaMalloc(&flush, fbytes);
  int hs[kBlocks], hd[kBlocks];
  // scattered: src = even-ish permutation of the low half, dst in the high half
  for (int i = 0; i < kBlocks; ++i) { hs[i] = (i * 37) % 512; hd[i] = 512 + (i * 101) % 512; }
  int *sb, *db; cudaMalloc(&sb, sizeof hs); cudaMalloc(&db, sizeof hd);
  cudaMemcpy(sb, hs, sizeof hs, cudaMemcpyHostToDevice); cudaMemcpy(db, hd, sizeof hd, cudaMemcpyHostToDevice);
  Args a{p, p, sb, db, plane, kPlanes * kBlocks * kTpp};
  cudaStream_t st; cudaStreamCreate(&st);
  bench("plain 256x8 (current)", copy_plain<256, 1>, 256, a, st, flush, fbytes);
  bench("plain 256x8 minblocks 6", copy_plain<256, 6>, 256, a, st, flush, fbytes);
  bench("plain 512x4", copy_plain<512, 1>, 512, a, st, flush, fbytes);
  bench("plain 1024x2", copy_plain<1024, 1>, 1024, a, st, flush, fbytes);
  bench("plain 128x16", copy_plain<128, 1>, 128, a, st, flush, fbytes);
  bench("pipe 256x8", copy_pipe<256>, 256, a, st, flush, fbytes);
  bench("pipe 512x4", copy_pipe<512>, 512, a, st, flush, fbytes);
  bench("pipe 1024x2", copy_pipe<1024>, 1024, a, st, flush, fbytes);
  // bulk reference point: cudaMemcpyAsync of one contiguous 2 GiB
  {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const size_t n = (size_t)kPlanes * kBlocks * kPiece;
    cudaMemcpyAsync(p + n, p, n, cudaMemcpyDeviceToDevice, st);
    cudaEventRecord(e0, st);
    cudaMemcpyAsync(p + n, p, n, cudaMemcpyDeviceToDevice, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s %8.1f us  %7.1f GB/s r+w\n", "cudaMemcpyAsync contiguous", ms * 1e3, 2.0 * n / ms / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
