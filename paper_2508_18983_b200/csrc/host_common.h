// host_common.h — host-side error plumbing shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <exception>
#include <string>

namespace moeb {

// Thrown inside the library; converted to a status code at the C boundary.
struct Error : std::exception {
  int code;
  std::string msg;
  Error(int c, std::string m) : code(c), msg(std::move(m)) {}
  const char* what() const noexcept override { return msg.c_str(); }
};

void set_last_error(const std::string& msg);

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(5, std::string(what) + ": " + cudaGetErrorString(e));
}
#define MOEB_CUDA(x) ::moeb::cuda_check((x), #x)

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    set_last_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return 4;
  }
}

// RAII device buffer.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  void alloc(size_t count) {
    free();
    n = count;
    if (count) MOEB_CUDA(cudaMalloc(&p, count * sizeof(T)));
  }
  void zero(cudaStream_t s = 0) {
    if (n) MOEB_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void free() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { free(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

}  // namespace moeb
