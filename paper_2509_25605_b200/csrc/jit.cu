// jit.cu — run-time compilation of generated kernels (the emitted Kokkos
// nests that have no hand-written kernel; paper_2509_25605_b200/cudagen.py).
//
// The reference compiles its emitted C++ ahead of time against Kokkos
// (emitter.py:596-780 -> g++ / Kokkos); here the executor
// (paper_2509_25605_b200/runtime.py) emits CUDA C++ for one nest at a time and
// this translation unit compiles it for sm_100a with NVRTC, loads the cubin
// with the runtime's library API and launches it.  NVRTC is dlopen'ed on first
// use so that loading liblapis_b200.so never needs it.  Compiled kernels are
// cached per (device, source): a program that runs the same nest again pays
// one hash lookup.
#include "common.cuh"

#include <dlfcn.h>

#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

namespace lapis_b200 {
namespace {

// --- the slice of the NVRTC API we use (nvrtc.h, resolved at run time)
typedef int nvrtcResult_t;
typedef struct _nvrtcProgram* nvrtcProgram_t;
struct Nvrtc {
  nvrtcResult_t (*create)(nvrtcProgram_t*, const char*, const char*, int, const char* const*,
                          const char* const*) = nullptr;
  nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char* const*) = nullptr;
  nvrtcResult_t (*log_size)(nvrtcProgram_t, size_t*) = nullptr;
  nvrtcResult_t (*log)(nvrtcProgram_t, char*) = nullptr;
  nvrtcResult_t (*cubin_size)(nvrtcProgram_t, size_t*) = nullptr;
  nvrtcResult_t (*cubin)(nvrtcProgram_t, char*) = nullptr;
  nvrtcResult_t (*destroy)(nvrtcProgram_t*) = nullptr;
  const char* (*error_string)(nvrtcResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

Nvrtc& nvrtc() {
  static Nvrtc api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnvrtc.so.12", "libnvrtc.so",
                           "/usr/local/cuda/lib64/libnvrtc.so.12"};
    void* h = nullptr;
    for (const char* n : names)
      if ((h = dlopen(n, RTLD_NOW | RTLD_LOCAL)) != nullptr) break;
    if (!h) {
      api.why = std::string("cannot load NVRTC: ") + dlerror();
      return;
    }
#define LB_SYM(field, sym)                                                   \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, sym));         \
  if (!api.field) {                                                          \
    api.why = std::string("NVRTC symbol missing: ") + sym;                   \
    return;                                                                  \
  }
    LB_SYM(create, "nvrtcCreateProgram");
    LB_SYM(compile, "nvrtcCompileProgram");
    LB_SYM(log_size, "nvrtcGetProgramLogSize");
    LB_SYM(log, "nvrtcGetProgramLog");
    LB_SYM(cubin_size, "nvrtcGetCUBINSize");
    LB_SYM(cubin, "nvrtcGetCUBIN");
    LB_SYM(destroy, "nvrtcDestroyProgram");
    LB_SYM(error_string, "nvrtcGetErrorString");
#undef LB_SYM
    api.ok = true;
  });
  return api;
}

struct Entry {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kernel = nullptr;
};

std::mutex g_mu;
std::unordered_map<std::string, Entry> g_cache;  // key: device '\0' name '\0' source

// NVRTC -> cubin for sm_100a.  --fmad=false keeps every mul and add separately
// rounded, the reference's per-op rounding (interp.py:168-171, and the
// -ffp-contract=off build of its emitted C++), so generated kernels are exact.
int compile_cubin(const char* source, const char* name, std::vector<char>& cubin) {
  Nvrtc& api = nvrtc();
  if (!api.ok) return fail(LAPIS_B200_ERR_UNSUPPORTED, api.why);
  nvrtcProgram_t prog = nullptr;
  nvrtcResult_t rc = api.create(&prog, source, name, 0, nullptr, nullptr);
  if (rc != 0) return fail(LAPIS_B200_ERR_CUDA, std::string("nvrtcCreateProgram: ") + api.error_string(rc));
  const char* opts[] = {"-arch=sm_100a", "--fmad=false", "-std=c++17", "-lineinfo",
                        "--device-as-default-execution-space"};
  rc = api.compile(prog, sizeof(opts) / sizeof(opts[0]), opts);
  if (rc != 0) {
    size_t n = 0;
    api.log_size(prog, &n);
    std::string log(n, '\0');
    if (n) api.log(prog, &log[0]);
    api.destroy(&prog);
    return fail(LAPIS_B200_ERR_ARG, std::string("NVRTC compile of ") + name + " failed:\n" + log);
  }
  size_t n = 0;
  api.cubin_size(prog, &n);
  cubin.resize(n);
  api.cubin(prog, cubin.data());
  api.destroy(&prog);
  return LAPIS_B200_OK;
}

}  // namespace
}  // namespace lapis_b200

using namespace lapis_b200;

extern "C" {

int lapis_b200_jit_available(void) { return nvrtc().ok ? 1 : 0; }

int lapis_b200_jit_compile(const char* source, const char* kernel_name, void** out_kernel) {
  if (!source || !kernel_name || !out_kernel) return fail(LAPIS_B200_ERR_ARG, "jit_compile: null argument");
  int dev = 0;
  LB_TRY(check_cuda(cudaGetDevice(&dev), "cudaGetDevice"));
  std::string key = std::to_string(dev);
  key.push_back('\0');
  key += kernel_name;
  key.push_back('\0');
  key += source;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_cache.find(key);
    if (it != g_cache.end()) {
      *out_kernel = reinterpret_cast<void*>(it->second.kernel);
      return LAPIS_B200_OK;
    }
  }
  std::vector<char> cubin;
  LB_TRY(compile_cubin(source, kernel_name, cubin));
  Entry e;
  LB_TRY(check_cuda(cudaLibraryLoadData(&e.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0),
                    "cudaLibraryLoadData"));
  cudaError_t ce = cudaLibraryGetKernel(&e.kernel, e.lib, kernel_name);
  if (ce != cudaSuccess) {
    cudaLibraryUnload(e.lib);
    return check_cuda(ce, "cudaLibraryGetKernel");
  }
  std::lock_guard<std::mutex> lk(g_mu);
  auto ins = g_cache.emplace(key, e);
  if (!ins.second) cudaLibraryUnload(e.lib);  // another thread won the race
  *out_kernel = reinterpret_cast<void*>(ins.first->second.kernel);
  return LAPIS_B200_OK;
}

// One by-value parameter block (the generated kernels take a single struct of
// 8-byte slots), grid-stride kernels so grid_x is a launch-size choice only.
int lapis_b200_jit_launch(void* kernel, int64_t grid_x, int block_x, int smem_bytes,
                          const void* params, int64_t params_bytes, void* stream) {
  if (!kernel) return fail(LAPIS_B200_ERR_ARG, "jit_launch: null kernel");
  if (grid_x <= 0 || grid_x > 0x7fffffff || block_x <= 0 || block_x > 1024)
    return fail(LAPIS_B200_ERR_ARG, "jit_launch: bad launch shape");
  if (params_bytes < 0 || params_bytes > 32000 || (params_bytes > 0 && !params))
    return fail(LAPIS_B200_ERR_ARG, "jit_launch: bad parameter block");
  void* args[1] = {const_cast<void*>(params)};
  cudaError_t e = cudaLaunchKernel(reinterpret_cast<const void*>(kernel), dim3((unsigned)grid_x),
                                   dim3((unsigned)block_x), params_bytes > 0 ? args : nullptr,
                                   (size_t)smem_bytes, reinterpret_cast<cudaStream_t>(stream));
  return check_cuda(e, "jit kernel launch");
}

// Compile only (no device needed): the build-time check of generated sources.
int lapis_b200_jit_check(const char* source, const char* kernel_name, int64_t* cubin_bytes) {
  if (!source || !kernel_name) return fail(LAPIS_B200_ERR_ARG, "jit_check: null argument");
  std::vector<char> cubin;
  LB_TRY(compile_cubin(source, kernel_name, cubin));
  if (cubin_bytes) *cubin_bytes = (int64_t)cubin.size();
  return LAPIS_B200_OK;
}

int lapis_b200_jit_cache_size(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  return (int)g_cache.size();
}

}  // extern "C"
