// Per-thread device context: the CUDA stream every lcnn call of this host
// thread is ordered on, stream-ordered HBM allocation from the device's
// cudaMallocAsync pool (see DeviceBuffer in device.hpp for the reuse rules),
// and the status -> exception mapping of the C ABI.
#include "lcnn/device.hpp"

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "lcnn_cuda.h"

namespace lcnn {

namespace {

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(std::string(what) + ": " + cudaGetErrorString(e));
}

struct ThreadContext {
  cudaStream_t stream = nullptr;
  cudaStream_t external = nullptr;  // caller-provided stream, if any
  int device = -1;
};

thread_local ThreadContext g_ctx;

// Keep freed blocks cached in the device's default pool (the default release
// threshold of 0 would return them to the driver at every sync).
void ensure_pool(int dev) {
  static std::mutex mu;
  static std::uint64_t done = 0;  // bit per device
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 64 && (done >> dev) & 1) return;
  cudaMemPool_t pool;
  cuda_ok(cudaDeviceGetDefaultMemPool(&pool, dev), "cudaDeviceGetDefaultMemPool");
  std::uint64_t threshold = UINT64_MAX;
  cuda_ok(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold),
          "cudaMemPoolSetAttribute");
  if (dev < 64) done |= std::uint64_t{1} << dev;
}

ThreadContext& ctx() {
  int dev = 0;
  cuda_ok(cudaGetDevice(&dev), "cudaGetDevice");
  if (g_ctx.stream == nullptr || g_ctx.device != dev) {
    cuda_ok(cudaStreamCreateWithFlags(&g_ctx.stream, cudaStreamNonBlocking),
            "cudaStreamCreate");
    g_ctx.device = dev;
    g_ctx.external = nullptr;
    ensure_pool(dev);
  }
  return g_ctx;
}

std::size_t round_bytes(std::size_t b) {
  if (b < 256) return 256;
  if (b < (1u << 20)) {  // powers of two below 1 MiB
    std::size_t r = 256;
    while (r < b) r <<= 1;
    return r;
  }
  const std::size_t mb = 1u << 20;  // 1 MiB granules above
  return (b + mb - 1) / mb * mb;
}

int initial_precision() {
  const char* env = std::getenv("LCNN_DENSE_PRECISION");
  if (!env) return LCNN_PREC_FP32;
  if (std::strcmp(env, "tf32") == 0) return LCNN_PREC_TF32;
  if (std::strcmp(env, "3xtf32") == 0) return LCNN_PREC_3XTF32;
  return LCNN_PREC_FP32;
}

std::atomic<int> g_precision{initial_precision()};

}  // namespace

DeviceBuffer::DeviceBuffer(std::size_t bytes) {
  ThreadContext& c = ctx();
  device_ = c.device;
  stream_ = c.external ? c.external : c.stream;
  bytes_ = round_bytes(bytes);
  const cudaStream_t s = static_cast<cudaStream_t>(stream_);
  cudaError_t e = cudaMallocAsync(&ptr_, bytes_, s);
  if (e != cudaSuccess) {
    // out of memory with blocks cached in the pool: drain, trim, retry once
    cudaGetLastError();
    cudaDeviceSynchronize();
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device_) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    cuda_ok(cudaMallocAsync(&ptr_, bytes_, s), "cudaMallocAsync");
  }
}

void DeviceBuffer::release() noexcept {
  if (!ptr_ || !owned_) return;
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) return;  // runtime torn down: leak quietly
  const cudaStream_t cur = g_ctx.external ? g_ctx.external : g_ctx.stream;
  if (dev == device_ && g_ctx.device == device_ && cur == static_cast<cudaStream_t>(stream_) &&
      cudaFreeAsync(ptr_, cur) == cudaSuccess) {
    ptr_ = nullptr;
    return;
  }
  cudaGetLastError();
  // foreign thread / stream / device: cudaFree waits for the device first
  if (dev != device_) cudaSetDevice(device_);
  cudaFree(ptr_);
  if (dev != device_) cudaSetDevice(dev);
  cudaGetLastError();
  ptr_ = nullptr;
}

DeviceBuffer DeviceBuffer::borrow(void* ptr, std::size_t bytes) {
  DeviceBuffer b;
  b.ptr_ = ptr;
  b.bytes_ = bytes;
  b.owned_ = false;
  return b;
}

DeviceBuffer::~DeviceBuffer() { release(); }

DeviceBuffer::DeviceBuffer(DeviceBuffer&& o) noexcept
    : ptr_(o.ptr_), bytes_(o.bytes_), owned_(o.owned_), device_(o.device_), stream_(o.stream_) {
  o.ptr_ = nullptr;
  o.bytes_ = 0;
}

DeviceBuffer& DeviceBuffer::operator=(DeviceBuffer&& o) noexcept {
  if (this != &o) {
    release();
    ptr_ = o.ptr_;
    bytes_ = o.bytes_;
    owned_ = o.owned_;
    device_ = o.device_;
    stream_ = o.stream_;
    o.ptr_ = nullptr;
    o.bytes_ = 0;
  }
  return *this;
}

void* current_stream() {
  ThreadContext& c = ctx();
  return c.external ? c.external : c.stream;
}

void set_current_stream(void* stream) {
  ThreadContext& c = ctx();
  if (c.external == static_cast<cudaStream_t>(stream)) return;  // no change: stay async
  // drain the stream being left: the caller may read its results or destroy
  // it right after switching -- unless the stream being entered is capturing
  // a CUDA graph (a synchronize would invalidate the capture; the capturing
  // caller orders the two streams itself, e.g. torch.cuda.graph's
  // wait_stream)
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (!(stream &&
        cudaStreamIsCapturing(static_cast<cudaStream_t>(stream), &cs) == cudaSuccess &&
        cs != cudaStreamCaptureStatusNone))
    synchronize();
  c.external = static_cast<cudaStream_t>(stream);
}

void synchronize() {
  cuda_ok(cudaStreamSynchronize(static_cast<cudaStream_t>(current_stream())),
          "cudaStreamSynchronize");
}

void throw_status(int status) {
  const std::string msg = lcnn_last_error();
  switch (status) {
    case LCNN_ESHAPE: throw ShapeError(msg);
    case LCNN_EINDEX: throw IndexError(msg);
    case LCNN_ELAYOUT: throw LayoutError(msg);
    case LCNN_EPLAN: throw PlanError(msg);
    case LCNN_EFORMAT: throw FormatError(msg);
    case LCNN_EDOMAIN: throw DomainError(msg);
    case LCNN_EUNSUPPORTED: throw UnsupportedError(msg);
    case LCNN_EVALIDATION: throw ValidationError(msg);
    case LCNN_ECALIBRATION: throw CalibrationError(msg);
    default: throw Error(std::string(lcnn_status_name(status)) + ": " + msg);
  }
}

DeviceTensor4D::DeviceTensor4D(std::uint32_t n, std::uint32_t c, std::uint32_t h,
                               std::uint32_t w, Layout layout)
    : n_(n), c_(c), h_(h), w_(w), layout_(layout) {
  if (!n || !c || !h || !w) throw ShapeError("Tensor4D: all dims must be >= 1");
  if (std::uint64_t{n} * c * h * w > 0xffffffffull)
    throw ShapeError("Tensor4D: dim product overflows");
  buf_ = std::make_shared<DeviceBuffer>(size() * sizeof(float));
}

DeviceTensor4D DeviceTensor4D::wrap(float* data, std::uint32_t n, std::uint32_t c,
                                    std::uint32_t h, std::uint32_t w, Layout layout) {
  DeviceTensor4D d;
  d.n_ = n;
  d.c_ = c;
  d.h_ = h;
  d.w_ = w;
  d.layout_ = layout;
  d.buf_ = std::make_shared<DeviceBuffer>(
      DeviceBuffer::borrow(data, std::uint64_t{n} * c * h * w * sizeof(float)));
  return d;
}

DeviceTensor4D DeviceTensor4D::upload(const Tensor4D& t) {
  DeviceTensor4D d(t.n(), t.c(), t.h(), t.w(), t.layout());
  cuda_ok(cudaMemcpyAsync(d.data(), t.data(), t.size() * sizeof(float), cudaMemcpyHostToDevice,
                          static_cast<cudaStream_t>(current_stream())),
          "upload");
  return d;
}

Tensor4D DeviceTensor4D::download() const {
  Tensor4D t(n_, c_, h_, w_, layout_);
  cuda_ok(cudaMemcpyAsync(t.data(), data(), size() * sizeof(float), cudaMemcpyDeviceToHost,
                          static_cast<cudaStream_t>(current_stream())),
          "download");
  synchronize();
  return t;
}

DeviceMatrix::DeviceMatrix(std::uint32_t r, std::uint32_t c)
    : rows(r), cols(c),
      buf(std::make_shared<DeviceBuffer>(std::uint64_t{r} * c * sizeof(float) + 16)) {}

DeviceMatrix DeviceMatrix::upload(const Matrix& m) {
  DeviceMatrix d(m.rows, m.cols);
  if (!m.data.empty())
    cuda_ok(cudaMemcpyAsync(d.data(), m.data.data(), m.data.size() * sizeof(float),
                            cudaMemcpyHostToDevice, static_cast<cudaStream_t>(current_stream())),
            "upload");
  return d;
}

Matrix DeviceMatrix::download() const {
  Matrix m(rows, cols);
  if (!m.data.empty())
    cuda_ok(cudaMemcpyAsync(m.data.data(), data(), m.data.size() * sizeof(float),
                            cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(current_stream())),
            "download");
  synchronize();
  return m;
}

void set_dense_precision(int precision) { g_precision.store(precision); }
int dense_precision() { return g_precision.load(); }

}  // namespace lcnn
