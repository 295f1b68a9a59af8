// Kernel-class timing scopes (see profile.cu).
#pragma once

#include <cuda_runtime.h>

namespace mph {
namespace prof {

// kinds match MPH_PROF_* in include/morphling.h
bool enabled();
void set_enabled(bool on);

class Scope {
 public:
  Scope(int kind, cudaStream_t s, double bytes, double flops);
  ~Scope();
  Scope(const Scope&) = delete;
  Scope& operator=(const Scope&) = delete;

 private:
  int idx_;
  cudaStream_t s_;
};

}  // namespace prof
}  // namespace mph
