// liblq JIT: expressions outside the closed families compiled by NVRTC into
// straight-line sm_100a kernels (the lowering step before the path, SURVEY.md
// §8(f) item 1).  NVRTC is opened lazily with dlopen so liblq.so has no
// link-time dependency on it; cubins are loaded with the runtime library API
// (cudaLibraryLoadData), so no driver-API linkage either.
#include <dlfcn.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "lq.h"

namespace {

typedef int nvrtcResult_;
typedef struct _nvrtcProgram* nvrtcProgram_;
struct Nvrtc {
    nvrtcResult_ (*create)(nvrtcProgram_*, const char*, const char*, int, const char* const*, const char* const*);
    nvrtcResult_ (*compile)(nvrtcProgram_, int, const char* const*);
    nvrtcResult_ (*cubin_size)(nvrtcProgram_, size_t*);
    nvrtcResult_ (*cubin)(nvrtcProgram_, char*);
    nvrtcResult_ (*log_size)(nvrtcProgram_, size_t*);
    nvrtcResult_ (*log)(nvrtcProgram_, char*);
    nvrtcResult_ (*destroy)(nvrtcProgram_*);
    bool ok = false;
    std::string why;
};

Nvrtc g_nvrtc;
std::once_flag g_nvrtc_once;

void load_nvrtc() {
    const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12",
                           "/usr/local/cuda/lib64/libnvrtc.so"};
    void* h = nullptr;
    for (const char* n : names)
        if ((h = dlopen(n, RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) {
        g_nvrtc.why = "libnvrtc.so.12 not found";
        return;
    }
#define LQ_SYM(field, name)                                                    \
    g_nvrtc.field = reinterpret_cast<decltype(g_nvrtc.field)>(dlsym(h, name)); \
    if (!g_nvrtc.field) {                                                      \
        g_nvrtc.why = std::string("missing NVRTC symbol ") + name;             \
        return;                                                                \
    }
    LQ_SYM(create, "nvrtcCreateProgram")
    LQ_SYM(compile, "nvrtcCompileProgram")
    LQ_SYM(cubin_size, "nvrtcGetCUBINSize")
    LQ_SYM(cubin, "nvrtcGetCUBIN")
    LQ_SYM(log_size, "nvrtcGetProgramLogSize")
    LQ_SYM(log, "nvrtcGetProgramLog")
    LQ_SYM(destroy, "nvrtcDestroyProgram")
#undef LQ_SYM
    g_nvrtc.ok = true;
}

}  // namespace

struct lq_jit {
    cudaLibrary_t lib = nullptr;
    cudaKernel_t lattice = nullptr;   // lq_jit_lattice (may be null)
    cudaKernel_t tensor = nullptr;    // lq_jit_tensor (may be null)
    std::vector<char> cubin;
};

// error reporting shared with lq_api.cu
int lq_internal_fail(int code, const char* fmt, ...);

extern "C" {

int lq_jit_create(const char* source, const char* name, lq_jit** out, char* log, int64_t log_cap) {
    if (!source || !out) return lq_internal_fail(LQ_ERR_VALUE, "null JIT source");
    std::call_once(g_nvrtc_once, load_nvrtc);
    if (!g_nvrtc.ok) return lq_internal_fail(LQ_ERR_UNSUPPORTED, "NVRTC unavailable: %s", g_nvrtc.why.c_str());
    nvrtcProgram_ prog = nullptr;
    if (g_nvrtc.create(&prog, source, name ? name : "lq_jit.cu", 0, nullptr, nullptr) != 0)
        return lq_internal_fail(LQ_ERR_CUDA, "nvrtcCreateProgram failed");
    const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--fmad=true", "-lineinfo"};
    const int rc = g_nvrtc.compile(prog, 4, opts);
    size_t ls = 0;
    g_nvrtc.log_size(prog, &ls);
    std::string lg(ls + 1, '\0');
    if (ls) g_nvrtc.log(prog, &lg[0]);
    if (log && log_cap > 0) {
        strncpy(log, lg.c_str(), (size_t)log_cap - 1);
        log[log_cap - 1] = '\0';
    }
    if (rc != 0) {
        g_nvrtc.destroy(&prog);
        return lq_internal_fail(LQ_ERR_VALUE, "NVRTC compile failed: %.400s", lg.c_str());
    }
    lq_jit* j = new lq_jit();
    size_t cs = 0;
    g_nvrtc.cubin_size(prog, &cs);
    j->cubin.resize(cs);
    g_nvrtc.cubin(prog, j->cubin.data());
    g_nvrtc.destroy(&prog);
    cudaError_t e = cudaLibraryLoadData(&j->lib, j->cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
    if (e != cudaSuccess) {
        delete j;
        return lq_internal_fail(LQ_ERR_CUDA, "cudaLibraryLoadData: %s", cudaGetErrorString(e));
    }
    if (cudaLibraryGetKernel(&j->lattice, j->lib, "lq_jit_lattice") != cudaSuccess) j->lattice = nullptr;
    if (cudaLibraryGetKernel(&j->tensor, j->lib, "lq_jit_tensor") != cudaSuccess) j->tensor = nullptr;
    cudaGetLastError();
    *out = j;
    return LQ_OK;
}

int lq_jit_destroy(lq_jit* j) {
    if (!j) return LQ_OK;
    if (j->lib) cudaLibraryUnload(j->lib);
    delete j;
    return LQ_OK;
}

}  // extern "C"

// used by lq_api.cu
cudaKernel_t lq_jit_lattice_kernel(const lq_jit* j) { return j ? j->lattice : nullptr; }
cudaKernel_t lq_jit_tensor_kernel(const lq_jit* j) { return j ? j->tensor : nullptr; }
