// TMA delivery microbenchmark (sm_100a): how many bytes per second the
// tensor-memory accelerator moves into shared memory for the box shapes the
// implicit-GEMM convolutions use.  One CTA per SM; thread 0 issues the boxes
// of a stage into a 4-deep ring (mbarrier complete_tx), thread 32 "consumes"
// each stage as soon as it lands.  No MMA, no stores: pure operand delivery.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tma_bench scripts/tma_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                             \
    }                                                                      \
  } while (0)

constexpr int kMaxStages = 8;  // ring slots (Cfg::stages, default 4)
constexpr int kMaxBoxes = 16;

struct Cfg {
  CUtensorMap map;
  int rank;
  int nbox;               // boxes per stage
  uint32_t box_bytes;     // bytes one box writes
  int32_t start[kMaxBoxes][5];  // coordinates of box j at iteration 0
  int32_t step[5];        // per-iteration coordinate advance (wrapped by `wrap`)
  int32_t wrap[5];        // coordinate wraps (0 = none)
  int32_t cta_step[5];    // per-CTA offset
  int iters;
  int stages;  // 0 = 4
  const void* bulk_src;  // RANK 1: cp.async.bulk of box_bytes from bulk_src + v[0] * box_bytes
};

__device__ __forceinline__ uint32_t sa(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int RANK, int NBOX>
__global__ void __launch_bounds__(64, 1) tma_kernel(const __grid_constant__ Cfg c, uint64_t* sink) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kMaxStages], empty[kMaxStages];
  const int kStages = c.stages ? c.stages : 4;
  const uint32_t stage_bytes = c.nbox * c.box_bytes;
  const uint32_t stride = (stage_bytes + 1023) / 1024 * 1024;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // coordinates advance incrementally (one compare per dimension per box),
    // so the issuing thread is never the bottleneck being measured
    int32_t x[NBOX][5];
#pragma unroll
    for (int j = 0; j < NBOX; ++j)
#pragma unroll
      for (int d = 0; d < 5; ++d) {
        int32_t v = c.start[j][d] + c.cta_step[d] * static_cast<int32_t>(blockIdx.x);
        if (c.wrap[d]) v %= c.wrap[d];
        x[j][d] = v;
      }
    const CUtensorMap* map = &c.map;
    int s = 0, ph = 0;
    for (int it = 0; it < c.iters; ++it) {
      asm volatile(
          "{\n.reg .pred p;\nW0:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W0;\n}\n" ::"r"(
              sa(&empty[s])),
          "r"(ph ^ 1)
          : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])),
                   "r"(stage_bytes)
                   : "memory");
      uint8_t* dst = smem + s * stride;
#pragma unroll
      for (int j = 0; j < NBOX; ++j, dst += c.box_bytes) {
        int32_t* v = x[j];
        if (RANK == 1)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  sa(dst)),
              "l"(reinterpret_cast<const uint8_t*>(c.bulk_src) + static_cast<uint64_t>(v[0]) * c.box_bytes),
              "r"(c.box_bytes), "r"(sa(&full[s]))
              : "memory");
        else if (RANK == 2)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                  sa(dst)),
              "l"(map), "r"(sa(&full[s])), "r"(v[0]), "r"(v[1])
              : "memory");
        else if (RANK == 3)
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
                  sa(dst)),
              "l"(map), "r"(sa(&full[s])), "r"(v[0]), "r"(v[1]), "r"(v[2])
              : "memory");
        else if (RANK == 4)
          asm volatile(
              "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
                  sa(dst)),
              "l"(map), "r"(sa(&full[s])), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3])
              : "memory");
        else
          asm volatile(
              "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(
                  sa(dst)),
              "l"(map), "r"(sa(&full[s])), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4])
              : "memory");
#pragma unroll
        for (int d = 0; d < 5; ++d) {
          v[d] += c.step[d];
          if (c.wrap[d] && v[d] >= c.wrap[d]) v[d] -= c.wrap[d];
        }
      }
      if (++s == kStages) {
        s = 0;
        ph ^= 1;
      }
    }
  } else if (threadIdx.x == 32) {
    int s = 0, ph = 0;
    uint64_t acc = 0;
    for (int it = 0; it < c.iters; ++it) {
      asm volatile(
          "{\n.reg .pred p;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W1;\n}\n" ::"r"(
              sa(&full[s])),
          "r"(ph)
          : "memory");
      acc += smem[s * stride + (it & 127)];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
      if (++s == kStages) {
        s = 0;
        ph ^= 1;
      }
    }
    if (acc == 0x123456789ull) sink[blockIdx.x] = acc;
  }
}

static bool encode(CUtensorMap* m, void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                   const uint32_t* box, CUtensorMapSwizzle sw) {
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = 1;
    if (i + 1 < rank) st[i] = strides_bytes[i];
  }
  CUresult r = cuTensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, base, d, st, b, e,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
  return r == CUDA_SUCCESS;
}

typedef void (*KernFn)(Cfg, uint64_t*);

template <int R>
KernFn pick_nbox(int n) {
  switch (n) {
    case 1: return tma_kernel<R, 1>;
    case 2: return tma_kernel<R, 2>;
    case 4: return tma_kernel<R, 4>;
    case 8: return tma_kernel<R, 8>;
    default: return tma_kernel<R, 12>;
  }
}

static void run(const char* name, Cfg& c, uint64_t* sink) {
  const uint32_t stage = c.nbox * c.box_bytes;
  const uint32_t stride = (stage + 1023) / 1024 * 1024;
  const size_t smem = (c.stages ? c.stages : 4) * stride + 1024;
  KernFn k = c.rank == 1 ? pick_nbox<1>(c.nbox) : c.rank == 2 ? pick_nbox<2>(c.nbox)
             : (c.rank == 3 ? pick_nbox<3>(c.nbox)
                            : (c.rank == 4 ? pick_nbox<4>(c.nbox) : pick_nbox<5>(c.nbox)));
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int rep = 0; rep < 2; ++rep) k<<<148, 64, smem>>>(c, sink);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  const int reps = 5;
  for (int rep = 0; rep < reps; ++rep) k<<<148, 64, smem>>>(c, sink);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  const double bytes = 148.0 * c.iters * stage;
  const double gbs = bytes / (ms * 1e6);
  printf("%-44s stage %6u B  %8.3f ms  %8.1f GB/s  %6.1f B/clk/SM  %7.1f ns/stage\n", name, stage, ms,
         gbs, gbs * 1e9 / 148 / 1.965e9, ms * 1e6 / c.iters);
}

int main() {
  uint64_t* sink;
  CK(cudaMalloc(&sink, 148 * 8));
  // conv1 input, CHWN: N=128, W=H=227, C=3 (79 MB, L2-resident after warm-up)
  const uint64_t N = 128, W = 227, H = 227, C = 3;
  float* x;
  CK(cudaMalloc(&x, 3000ull * 256 * 128 + 4096));
  CK(cudaMemset(x, 0, 3000ull * 256 * 128));
  const int iters = 2000;
  auto zero = [](Cfg& c) { memset(&c, 0, sizeof(c)); };
  // TB_ONLY=conv4: only the conv3-5 input-box comparison at the end
  const bool only_c4 = getenv("TB_ONLY") != nullptr;
  if (only_c4) goto conv4_boxes;

  // A: the conv1 ROW box {32 n, 11 w, 1 h, 3 c}, 4 n-groups per stage, walks (ow, oh)
  for (int swz = 0; swz < 3; ++swz) {
    Cfg c;
    zero(c);
    const uint64_t dims[4] = {N, W, H, C};
    const uint64_t str[3] = {N * 4, W * N * 4, H * W * N * 4};
    const uint32_t box[4] = {32, 11, 1, 3};
    CUtensorMapSwizzle sw = swz == 0 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                                     : (swz == 1 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE);
    encode(&c.map, x, 4, dims, str, box, sw);
    c.rank = 4;
    c.nbox = 4;
    c.box_bytes = 32 * 11 * 3 * 4;
    for (int j = 0; j < 4; ++j) c.start[j][0] = 32 * j;
    c.step[1] = 4; c.wrap[1] = 216;   // ow * 4
    c.step[2] = 1; c.wrap[2] = 216;   // oh*4+fh
    c.cta_step[1] = 4; c.cta_step[2] = 1;
    c.iters = iters;
    run(swz == 0 ? "conv1 box{32,11,1,3} x4  ATOM_32B" : (swz == 1 ? "conv1 box{32,11,1,3} x4  SW128" : "conv1 box{32,11,1,3} x4  NONE"), c, sink);
  }
  // B: per channel boxes {32, 11, 1, 1} x 3 c x 4 n
  {
    Cfg c;
    zero(c);
    const uint64_t dims[4] = {N, W, H, C};
    const uint64_t str[3] = {N * 4, W * N * 4, H * W * N * 4};
    const uint32_t box[4] = {32, 11, 1, 1};
    encode(&c.map, x, 4, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    c.rank = 4;
    c.nbox = 12;
    c.box_bytes = 32 * 11 * 4;
    for (int j = 0; j < 12; ++j) {
      c.start[j][0] = 32 * (j % 4);
      c.start[j][3] = j / 4;
    }
    c.step[1] = 4; c.wrap[1] = 216;
    c.step[2] = 1; c.wrap[2] = 216;
    c.cta_step[1] = 4; c.cta_step[2] = 1;
    c.iters = iters;
    run("conv1 box{32,11,1,1} x12 ATOM_32B", c, sink);
  }
  // C: 5D map folding the 4 n-groups: {32, 4, W, H, C}, box {32, 4, 11, 1, 3}
  {
    Cfg c;
    zero(c);
    const uint64_t dims[5] = {32, 4, W, H, C};
    const uint64_t str[4] = {128, N * 4, W * N * 4, H * W * N * 4};
    const uint32_t box[5] = {32, 4, 11, 1, 3};
    encode(&c.map, x, 5, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    c.rank = 5;
    c.nbox = 1;
    c.box_bytes = 32 * 4 * 11 * 3 * 4;
    c.step[2] = 4; c.wrap[2] = 216;
    c.step[3] = 1; c.wrap[3] = 216;
    c.cta_step[2] = 4; c.cta_step[3] = 1;
    c.iters = iters;
    run("conv1 5D box{32,4,11,1,3} x1 ATOM_32B", c, sink);
  }
  // D: a 2D view of the same bytes: rows of 128 floats (one pixel x 128 n), box {32, 33}
  {
    Cfg c;
    zero(c);
    const uint64_t rows = W * H * C;
    const uint64_t dims[2] = {N, rows};
    const uint64_t str[1] = {N * 4};
    const uint32_t box[2] = {32, 33};
    encode(&c.map, x, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    c.rank = 2;
    c.nbox = 4;
    c.box_bytes = 32 * 33 * 4;
    for (int j = 0; j < 4; ++j) c.start[j][0] = 32 * j;
    c.step[1] = 4; c.wrap[1] = 150000;
    c.cta_step[1] = 1000;
    c.iters = iters;
    run("2D box{32,33} x4 (contiguous rows) ATOM_32B", c, sink);
  }
  // E: 2D GEMM-B-like: [K=9216][N=4096] fp32, box {32 n, 32 k} x 8 (32 KB)
  {
    Cfg c;
    zero(c);
    const uint64_t dims[2] = {4096, 4608};
    const uint64_t str[1] = {4096 * 4};
    const uint32_t box[2] = {32, 32};
    encode(&c.map, x, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    c.rank = 2;
    c.nbox = 8;
    c.box_bytes = 32 * 32 * 4;
    for (int j = 0; j < 8; ++j) c.start[j][0] = 32 * j;
    c.step[1] = 32; c.wrap[1] = 4576;
    c.cta_step[0] = 256; c.wrap[0] = 4096;
    c.iters = iters;
    run("gemm-B box{32,32} x8 ATOM_32B", c, sink);
  }
  // F: 2D GEMM-A-like K-major: [M][K], box {32 k, 128 m} SW128
  {
    Cfg c;
    zero(c);
    const uint64_t dims[2] = {4096, 4608};
    const uint64_t str[1] = {4096 * 4};
    const uint32_t box[2] = {32, 128};
    encode(&c.map, x, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
    c.rank = 2;
    c.nbox = 2;
    c.box_bytes = 32 * 128 * 4;
    c.start[1][1] = 128;
    c.step[0] = 32; c.wrap[0] = 4064;
    c.cta_step[1] = 256; c.wrap[1] = 4352;
    c.iters = iters;
    run("gemm-A box{32,128} x2 SW128", c, sink);
  }
  // G: conv2 CI box: input N=128, 27x27, C=96, box {32, 1, 1, 32} x 4
  {
    Cfg c;
    zero(c);
    const uint64_t W2 = 27, H2 = 27, C2 = 96;
    const uint64_t dims[4] = {N, W2, H2, C2};
    const uint64_t str[3] = {N * 4, W2 * N * 4, H2 * W2 * N * 4};
    const uint32_t box[4] = {32, 1, 1, 32};
    encode(&c.map, x, 4, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    c.rank = 4;
    c.nbox = 4;
    c.box_bytes = 32 * 32 * 4;
    for (int j = 0; j < 4; ++j) c.start[j][0] = 32 * j;
    c.step[1] = 1; c.wrap[1] = 27;
    c.step[3] = 32; c.wrap[3] = 96;
    c.cta_step[2] = 1; c.wrap[2] = 27;
    c.iters = iters;
    run("conv2 CI box{32,1,1,32} x4 ATOM_32B", c, sink);
  }
  // H: conv2 5D folding n-groups {32, 4, W, H, C} box {32, 4, 1, 1, 32}
  {
    Cfg c;
    zero(c);
    const uint64_t W2 = 27, H2 = 27, C2 = 96;
    const uint64_t dims[5] = {32, 4, W2, H2, C2};
    const uint64_t str[4] = {128, N * 4, W2 * N * 4, H2 * W2 * N * 4};
    const uint32_t box[5] = {32, 4, 1, 1, 32};
    encode(&c.map, x, 5, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    c.rank = 5;
    c.nbox = 1;
    c.box_bytes = 32 * 4 * 32 * 4;
    c.step[2] = 1; c.wrap[2] = 27;
    c.step[4] = 32; c.wrap[4] = 96;
    c.cta_step[3] = 1; c.wrap[3] = 27;
    c.iters = iters;
    run("conv2 5D box{32,4,1,1,32} x1 ATOM_32B", c, sink);
  }
  // I: fc-B grouped 3D view {32 n, K, N/32 groups} (group stride 128 B < k stride), box {32, 32, 8}
  {
    Cfg c;
    zero(c);
    const uint64_t dims[3] = {32, 4608, 128};
    const uint64_t str[2] = {4096 * 4, 128};
    const uint32_t box[3] = {32, 32, 8};
    if (encode(&c.map, x, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) {
      c.rank = 3;
      c.nbox = 1;
      c.box_bytes = 32 * 32 * 8 * 4;
      c.step[1] = 32; c.wrap[1] = 4576;
      c.cta_step[2] = 8; c.wrap[2] = 128;
      c.iters = iters;
      run("fc-B grouped 3D box{32,32,8} x1", c, sink);
    }
  }
  // J: conv2 CI grouped 5D view {32 n, C, G, W, H}, box {32, 32 c, 4 g, 1, 1}
  {
    Cfg c;
    zero(c);
    const uint64_t W2 = 27, H2 = 27, C2 = 96;
    const uint64_t dims[5] = {32, C2, 4, W2, H2};
    const uint64_t str[4] = {H2 * W2 * N * 4, 128, N * 4, W2 * N * 4};
    const uint32_t box[5] = {32, 32, 4, 1, 1};
    if (encode(&c.map, x, 5, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) {
      c.rank = 5;
      c.nbox = 2;
      c.box_bytes = 32 * 32 * 4 * 4;
      c.start[1][3] = 1;
      c.step[1] = 32; c.wrap[1] = 96;
      c.step[3] = 1; c.wrap[3] = 26;
      c.cta_step[4] = 1; c.wrap[4] = 27;
      c.iters = iters;
      run("conv2 grouped 5D box{32,32,4,1,1} x2", c, sink);
    }
  }
  // K: conv1 grouped 5D view {32 n, W, C, G, H}, box {32, 16 w, 3 c, 4 g, 1}, 2 pixels
  {
    Cfg c;
    zero(c);
    const uint64_t dims[5] = {32, W, C, 4, H};
    const uint64_t str[4] = {N * 4, H * W * N * 4, 128, W * N * 4};
    const uint32_t box[5] = {32, 16, 3, 4, 1};
    if (encode(&c.map, x, 5, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) {
      c.rank = 5;
      c.nbox = 2;
      c.box_bytes = 32 * 16 * 3 * 4 * 4;
      c.start[1][1] = 4;
      c.step[1] = 8; c.wrap[1] = 208;
      c.step[4] = 1; c.wrap[4] = 216;
      c.cta_step[1] = 8; c.cta_step[4] = 1;
      c.iters = iters;
      run("conv1 grouped 5D box{32,16,3,4,1} x2", c, sink);
    }
  }
  // N: contiguous weight images: 1D bulk copies vs a 2D tensor box over the
  // same bytes ([rows][32] floats, pitch 128 B), 24 KB (192 rows) and 32 KB
  for (int rows : {192, 256}) {
    Cfg c;
    zero(c);
    c.rank = 1;
    c.nbox = 1;
    c.box_bytes = rows * 128;
    c.bulk_src = x;
    c.step[0] = 1; c.wrap[0] = 3000;
    c.cta_step[0] = 20;
    c.iters = iters;
    char name[64];
    snprintf(name, sizeof(name), "bulk 1D %d KB", rows / 8);
    run(name, c, sink);
    Cfg d;
    zero(d);
    const uint64_t dims[2] = {32, 3000ull * rows};
    const uint64_t str[1] = {128};
    const uint32_t box[2] = {32, (uint32_t)rows};
    if (encode(&d.map, x, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) {
      d.rank = 2;
      d.nbox = 1;
      d.box_bytes = rows * 128;
      d.step[1] = rows; d.wrap[1] = 2990 * rows;
      d.cta_step[1] = 20 * rows;
      d.iters = iters;
      snprintf(name, sizeof(name), "2D box{32,%d} contiguous SW128", rows);
      run(name, d, sink);
    }
    // the strided original: box {32 k, rows} over a [rows][K] matrix with K = 2400
    Cfg e;
    zero(e);
    const uint64_t dims2[2] = {2400, 1536};
    const uint64_t str2[1] = {2400 * 4};
    const uint32_t box2[2] = {32, (uint32_t)rows};
    if (encode(&e.map, x, 2, dims2, str2, box2, CU_TENSOR_MAP_SWIZZLE_128B)) {
      e.rank = 2;
      e.nbox = 1;
      e.box_bytes = rows * 128;
      e.step[0] = 32; e.wrap[0] = 2400;
      e.cta_step[1] = rows; e.wrap[1] = 1536 - rows;
      e.iters = iters;
      snprintf(name, sizeof(name), "2D box{32,%d} strided K=2400 SW128", rows);
      run(name, e, sink);
    }
  }
  // L: conv1 SHARE box: view {32 n, C, W, G, H} (rows ordered (w, c)), box
  // {32, 3 c, 39 w, 1 g, 1 h}: 8 output pixels of one 32-image group per box
  for (int slots : {3, 4, 6, 8}) {
    Cfg c;
    zero(c);
    const uint64_t dims[5] = {32, C, W, 4, H};
    const uint64_t str[4] = {H * W * N * 4, N * 4, 128, W * N * 4};
    const uint32_t box[5] = {32, 3, 39, 1, 1};
    if (encode(&c.map, x, 5, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) {
      c.rank = 5;
      c.nbox = 1;
      c.box_bytes = 32 * 3 * 39 * 4;
      c.step[4] = 1; c.wrap[4] = 216;   // filter rows / output rows
      c.cta_step[2] = 32; c.wrap[2] = 190;
      c.cta_step[3] = 1; c.wrap[3] = 4;
      c.iters = iters;
      c.stages = slots;
      char name[64];
      snprintf(name, sizeof(name), "conv1 SHARE box{32,3,39,1,1} x1 slots=%d", slots);
      run(name, c, sink);
    }
  }
  // M: same, 2 boxes per stage (2 groups)
  {
    Cfg c;
    zero(c);
    const uint64_t dims[5] = {32, C, W, 4, H};
    const uint64_t str[4] = {H * W * N * 4, N * 4, 128, W * N * 4};
    const uint32_t box[5] = {32, 3, 39, 1, 1};
    if (encode(&c.map, x, 5, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) {
      c.rank = 5;
      c.nbox = 2;
      c.box_bytes = 32 * 3 * 39 * 4;
      c.start[1][3] = 1;
      c.step[4] = 1; c.wrap[4] = 216;
      c.cta_step[2] = 32; c.wrap[2] = 190;
      c.iters = iters;
      c.stages = 4;
      run("conv1 SHARE box x2 (2 groups) slots=4", c, sink);
    }
  }
  if (getenv("TB_BLK")) goto blocked_boxes;
  if (getenv("TB_VGG")) goto vgg_boxes;
conv4_boxes:
  // P/Q/R: AlexNet conv4 input (N=128, 13x13, C=384, CHWN: 33 MB, L2-resident),
  // the CI k-block of a RowsOut tile: 32 channels x 2 output pixels x 128 images.
  {
    const uint64_t W4 = 13, H4 = 13, C4 = 384, plane = H4 * W4 * N * 4;
    // P: shipped grouped 5D view {32 n, C, 4 g, W, H}, box {32, 32 c, 4 g, 1, 1} x 2 pixels
    {
      Cfg c;
      zero(c);
      const uint64_t dims[5] = {32, C4, 4, W4, H4};
      const uint64_t str[4] = {plane, 128, N * 4, W4 * N * 4};
      const uint32_t box[5] = {32, 32, 4, 1, 1};
      if (encode(&c.map, x, 5, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) {
        c.rank = 5; c.nbox = 2; c.box_bytes = 32 * 32 * 4 * 4;
        c.start[1][3] = 1;
        c.step[1] = 32; c.wrap[1] = 384;
        c.step[3] = 2; c.wrap[3] = 12;
        c.cta_step[4] = 1; c.wrap[4] = 13;
        c.iters = iters;
        run("conv4 grouped 5D box{32,32,4,1,1} x2", c, sink);
      }
    }
    // Q: (w, g) merged into one dim of stride 128 B: 4D view {32 n, C, 4W, H},
    // ONE box {32, 32 c, 8, 1} lands both pixels' 8 atoms in the same order
    for (int nb : {1, 2}) {
      Cfg c;
      zero(c);
      const uint64_t dims[4] = {32, C4, 4 * W4, H4};
      const uint64_t str[3] = {plane, 128, W4 * N * 4};
      const uint32_t box[4] = {32, 32, (uint32_t)(8 / nb), 1};
      if (encode(&c.map, x, 4, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) {
        c.rank = 4; c.nbox = nb; c.box_bytes = 32 * 32 * (8 / nb) * 4;
        if (nb == 2) c.start[1][2] = 4;
        c.step[1] = 32; c.wrap[1] = 384;
        c.step[2] = 8; c.wrap[2] = 48;
        c.cta_step[3] = 1; c.wrap[3] = 13;
        c.iters = iters;
        run(nb == 1 ? "conv4 merged 4D box{32,32,8,1} x1" : "conv4 merged 4D box{32,32,4,1} x2", c, sink);
      }
    }
    // R: the filter tile of the same stage, K-major [Co=256][K=3456], box {32 k, 128 co}
    {
      Cfg c;
      zero(c);
      const uint64_t dims[2] = {3456, 256};
      const uint64_t str[1] = {3456 * 4};
      const uint32_t box[2] = {32, 128};
      if (encode(&c.map, x, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) {
        c.rank = 2; c.nbox = 1; c.box_bytes = 32 * 128 * 4;
        c.step[0] = 32; c.wrap[0] = 3456;
        c.cta_step[1] = 128; c.wrap[1] = 256;
        c.iters = iters;
        run("conv4 filter box{32,128} K-major SW128", c, sink);
      }
    }
  }
  return 0;
vgg_boxes:
  // S/T: VGG conv1_2 input (N=128, 224x224, C=64, CHWN: 1.64 GB, DRAM-cold),
  // the TAPS input box of one (filter row, 32-channel block):
  //  S: shipped, 8 pixels x 32 images: view {32 n, C, W, 4 g, H}, box {32, 32 c, 10 w, 1, 1}
  //     (40 KB: 320 runs of 128 B, one 32-image group per CTA, 4 CTAs per pixel block)
  //  T: 2 pixels x 128 images: view {32 n, C, 4 g, W, H}, box {32, 32 c, 4 g, 4 w, 1}
  //     (64 KB: per channel 2 KB contiguous -- 4 pixels x 4 groups -- in one box)
  {
    const uint64_t Nv = 128, Wv = 224, Hv = 224, Cv = 64, plane = Hv * Wv * Nv * 4;
    float* xv;
    CK(cudaMalloc(&xv, plane * Cv + 4096));
    CK(cudaMemset(xv, 0, plane * Cv));
    for (int st : {3, 4}) {
      Cfg c;
      zero(c);
      const uint64_t dims[5] = {32, Cv, Wv, 4, Hv};
      const uint64_t str[4] = {plane, Nv * 4, 128, Wv * Nv * 4};
      const uint32_t box[5] = {32, 32, 10, 1, 1};
      if (encode(&c.map, xv, 5, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) {
        c.rank = 5; c.nbox = 1; c.box_bytes = 32 * 32 * 10 * 4; c.stages = st;
        c.step[1] = 32; c.wrap[1] = 64;
        c.step[4] = 1; c.wrap[4] = 222;
        c.cta_step[3] = 1; c.wrap[3] = 4;
        c.cta_step[2] = 2; c.wrap[2] = 210;
        c.iters = 1500;
        run(st == 3 ? "vgg1_2 TAPS box{32,32,10,1,1} 3 slots" : "vgg1_2 TAPS box{32,32,10,1,1} 4 slots", c, sink);
      }
    }
    for (int st : {2, 3}) {
      Cfg c;
      zero(c);
      const uint64_t dims[5] = {32, Cv, 4, Wv, Hv};
      const uint64_t str[4] = {plane, 128, Nv * 4, Wv * Nv * 4};
      const uint32_t box[5] = {32, 32, 4, 4, 1};
      if (encode(&c.map, xv, 5, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) {
        c.rank = 5; c.nbox = 1; c.box_bytes = 32 * 32 * 4 * 4 * 4; c.stages = st;
        c.step[1] = 32; c.wrap[1] = 64;
        c.step[4] = 1; c.wrap[4] = 222;
        c.cta_step[3] = 3; c.wrap[3] = 219;
        c.iters = 1500;
        run(st == 2 ? "vgg1_2 wide box{32,32,4,4,1} 2 slots" : "vgg1_2 wide box{32,32,4,4,1} 3 slots", c, sink);
      }
    }
    CK(cudaFree(xv));
  }
  // U: the same TAPS box with the channel-plane pitch padded (plane + pad bytes): are the 32
  // rows of one box, a plane (a multiple of 512 KB) apart, camping on the same L2 slice / DRAM
  // bank?  DRAM-cold (224 rows) and L2-resident (8 rows, 58 MB) versions.
  {
    const uint64_t Nv = 128, Wv = 224, Cv = 64;
    for (uint64_t Hv : {224ull, 8ull}) {
      for (uint64_t pad : {0ull, 128ull, 1152ull, 4224ull}) {
        if (Hv == 8 && (pad == 128 || pad == 4224)) continue;
        const uint64_t plane = Hv * Wv * Nv * 4 + pad;
        float* xv;
        CK(cudaMalloc(&xv, plane * Cv + 4096));
        CK(cudaMemset(xv, 0, plane * Cv));
        Cfg c;
        zero(c);
        const uint64_t dims[5] = {32, Cv, Wv, 4, Hv};
        const uint64_t str[4] = {plane, Nv * 4, 128, Wv * Nv * 4};
        const uint32_t box[5] = {32, 32, 10, 1, 1};
        if (encode(&c.map, xv, 5, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) {
          c.rank = 5; c.nbox = 1; c.box_bytes = 32 * 32 * 10 * 4; c.stages = 3;
          c.step[1] = 32; c.wrap[1] = 64;
          c.step[4] = 1; c.wrap[4] = (int)Hv - 2;
          c.cta_step[3] = 1; c.wrap[3] = 4;
          c.cta_step[2] = 2; c.wrap[2] = 210;
          c.iters = Hv == 8 ? 3000 : 1500;
          char name[96];
          snprintf(name, sizeof name, "vgg1_2 TAPS box H=%llu plane pad %llu B", (unsigned long long)Hv,
                   (unsigned long long)pad);
          run(name, c, sink);
        }
        CK(cudaFree(xv));
      }
    }
  }
blocked_boxes:
  // V: the same TAPS box {32 n, 32 c, 10 w} of VGG conv1_2's input (N=128, C=64, 224 x 224)
  // over three HBM layouts of the same tensor, DRAM-cold (H=224) and L2-resident (H=8):
  //   CHWN           [c][h][w][n]      a (c, w) row is 128 B of a 512-B (c,h,w) line
  //   CHWN32 blocked [g][c][h][w][32]  a box row-run is 10 w x 128 B = 1280 B contiguous
  //   HWCN32 blocked [g][h][w][c][32]  a box is 10 runs of 32 c x 128 B = 4 KB contiguous
  {
    const uint64_t Nv = 128, Wv = 224, Cv = 64, G = Nv / 32;
    for (uint64_t Hv : {224ull, 8ull}) {
      const uint64_t bytes = Hv * Wv * Nv * 4 * Cv;
      float* xv;
      CK(cudaMalloc(&xv, bytes + 4096));
      CK(cudaMemset(xv, 0, bytes));
      for (int lay = 0; lay < 3; ++lay) {
        Cfg c;
        zero(c);
        // dims {32 n, C, W, G, H}; strides of c, w, g, h in bytes
        uint64_t str[4];
        if (lay == 0) {
          str[0] = Hv * Wv * Nv * 4; str[1] = Nv * 4; str[2] = 128; str[3] = Wv * Nv * 4;
        } else if (lay == 1) {
          str[0] = Hv * Wv * 128; str[1] = 128; str[2] = Cv * Hv * Wv * 128; str[3] = Wv * 128;
        } else {
          str[0] = 128; str[1] = Cv * 128; str[2] = Hv * Wv * Cv * 128; str[3] = Wv * Cv * 128;
        }
        const uint64_t dims[5] = {32, Cv, Wv, G, Hv};
        const uint32_t box[5] = {32, 32, 10, 1, 1};
        if (encode(&c.map, xv, 5, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) {
          c.rank = 5; c.nbox = 1; c.box_bytes = 32 * 32 * 10 * 4; c.stages = 3;
          c.step[1] = 32; c.wrap[1] = 64;
          c.step[4] = 1; c.wrap[4] = (int)Hv - 2;
          c.cta_step[3] = 1; c.wrap[3] = 4;
          c.cta_step[2] = 2; c.wrap[2] = 210;
          c.iters = Hv == 8 ? 3000 : 1500;
          char name[96];
          snprintf(name, sizeof name, "vgg1_2 TAPS box H=%llu layout %s", (unsigned long long)Hv,
                   lay == 0 ? "CHWN" : lay == 1 ? "CHWN32 blocked" : "HWCN32 blocked");
          run(name, c, sink);
        }
      }
      CK(cudaFree(xv));
    }
  }
  return 0;
}
