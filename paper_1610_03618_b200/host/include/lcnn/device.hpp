// Device-resident extension of the lcnn API (not in the reference): HBM
// buffers, a per-host-thread CUDA stream, and device overloads of the hot
// ops so whole networks run without host round trips.  Host-tensor calls in
// layout.hpp / pool.hpp / softmax.hpp / conv.hpp are thin wrappers: upload,
// one C-ABI kernel call (include/lcnn_cuda.h), download.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>

#include "lcnn/tensor.hpp"

namespace lcnn {

// Owning HBM allocation from the device's stream-ordered pool
// (cudaMallocAsync on the calling thread's current stream, with the pool's
// release threshold raised so freed blocks stay cached).  The buffer records
// its device and that stream: freed on the same thread context with the same
// current stream it is returned with cudaFreeAsync (ordered after every
// kernel queued there, never a sync); freed anywhere else (another host
// thread, another current stream or device) it is released with cudaFree,
// which waits for the device, so a block can never be reused while a kernel
// on its owner stream may still touch it.
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(std::size_t bytes);
  // Non-owning view of caller memory (never returned to the pool).
  static DeviceBuffer borrow(void* ptr, std::size_t bytes);
  ~DeviceBuffer();
  DeviceBuffer(DeviceBuffer&& o) noexcept;
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept;
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;

  float* f() const { return static_cast<float*>(ptr_); }
  void* get() const { return ptr_; }
  std::size_t bytes() const { return bytes_; }

 private:
  void release() noexcept;
  void* ptr_ = nullptr;
  std::size_t bytes_ = 0;
  bool owned_ = true;
  int device_ = -1;
  void* stream_ = nullptr;  // cudaStream_t the block was allocated on
};

// The stream every lcnn call issued from this host thread is ordered on.
void* current_stream();
// Order this thread's lcnn calls on a caller-owned stream (nullptr restores
// the library's own stream).
void set_current_stream(void* stream);
// Block until the calling thread's stream has drained.
void synchronize();
// Throw the lcnn exception matching a non-OK lcnn_status (with the library's
// message), e.g. PlanError for LCNN_EPLAN.
void throw_status(int status);
inline void check_status(int status) {
  if (status != 0) throw_status(status);
}

class DeviceTensor4D {
 public:
  DeviceTensor4D(std::uint32_t n, std::uint32_t c, std::uint32_t h,
                 std::uint32_t w, Layout layout);
  static DeviceTensor4D upload(const Tensor4D& t);
  // View of caller-owned device memory in the given layout (not copied).
  static DeviceTensor4D wrap(float* data, std::uint32_t n, std::uint32_t c, std::uint32_t h,
                             std::uint32_t w, Layout layout);
  Tensor4D download() const;

  std::uint32_t n() const { return n_; }
  std::uint32_t c() const { return c_; }
  std::uint32_t h() const { return h_; }
  std::uint32_t w() const { return w_; }
  Layout layout() const { return layout_; }
  void set_layout_tag(Layout l) { layout_ = l; }
  std::uint64_t size() const { return std::uint64_t{n_} * c_ * h_ * w_; }
  float* data() const { return buf_->f(); }
  const std::shared_ptr<DeviceBuffer>& buffer() const { return buf_; }

 private:
  DeviceTensor4D() = default;
  std::uint32_t n_ = 0, c_ = 0, h_ = 0, w_ = 0;
  Layout layout_ = Layout::NCHW;
  std::shared_ptr<DeviceBuffer> buf_;
};

struct DeviceMatrix {
  std::uint32_t rows = 0, cols = 0;
  std::shared_ptr<DeviceBuffer> buf;
  DeviceMatrix() = default;
  DeviceMatrix(std::uint32_t r, std::uint32_t c);
  static DeviceMatrix upload(const Matrix& m);
  Matrix download() const;
  float* data() const { return buf->f(); }
};

// Convolution / GEMM arithmetic of the host-tensor API (lcnn_precision
// codes) and the default a Network takes at construction.  Default FP32 keeps
// the reference's 1e-5 tolerances.  A Network resolves its precision once
// (RunOptions::dense_precision, else this default) and never reads the
// process default again, so networks at different precisions can run side
// by side on different threads.
void set_dense_precision(int precision);
int dense_precision();

}  // namespace lcnn
