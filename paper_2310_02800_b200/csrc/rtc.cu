// Runtime-specialised mining kernels: the paper's
// "code generator ... compiled into a shared library" per query (P:603-611,
// P:739-780), done with NVRTC.  tm_motif_specialise instantiates the same
// mine_kernel<PlanC<CODE, GEN>, MODE> template the build-time catalog uses —
// from the same headers, embedded at build time (build/rtc_sources.inc) — for
// any motif, and with GEN = true for motifs with labels / anti-edges.  The
// cubin is loaded through the driver API; one compile per (device, code,
// GEN, mode) per process.
#include <cuda.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "tm_internal.cuh"

namespace tmg {
namespace {

#include "rtc_sources.inc"   // kRtcInternal, kRtcMine, kRtcApiMacros (build.py)

struct Entry {
    CUmodule mod = nullptr;
    CUfunction fn = nullptr;
    int smem_per_warp = 0;
};

std::mutex g_mu;
std::map<std::tuple<int, uint64_t, bool, int>, Entry> g_cache;

// Driver API entry points through cudart (cudaGetDriverEntryPoint), so the
// library does not link libcuda and still loads on a machine without a driver.
struct Driver {
    CUresult (*GetErrorString)(CUresult, const char **) = nullptr;
    CUresult (*ModuleLoadData)(CUmodule *, const void *) = nullptr;
    CUresult (*ModuleGetFunction)(CUfunction *, CUmodule, const char *) = nullptr;
    CUresult (*ModuleGetGlobal)(CUdeviceptr *, size_t *, CUmodule, const char *) = nullptr;
    CUresult (*MemcpyDtoH)(void *, CUdeviceptr, size_t) = nullptr;
    CUresult (*FuncSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
    CUresult (*OccupancyMaxActiveBlocksPerMultiprocessor)(int *, CUfunction, int, size_t) = nullptr;
    CUresult (*LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                             CUstream, void **, void **) = nullptr;
    CUresult (*LaunchCooperativeKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                                        unsigned, CUstream, void **) = nullptr;
    bool ok = false;
};

template <class F>
bool entry(const char *name, F &f) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p) return false;
    f = reinterpret_cast<F>(p);
    return true;
}

const Driver &drv() {
    static Driver d = [] {
        Driver x;
        x.ok = entry("cuGetErrorString", x.GetErrorString) && entry("cuModuleLoadData", x.ModuleLoadData) &&
               entry("cuModuleGetFunction", x.ModuleGetFunction) && entry("cuModuleGetGlobal", x.ModuleGetGlobal) &&
               entry("cuMemcpyDtoH", x.MemcpyDtoH) && entry("cuFuncSetAttribute", x.FuncSetAttribute) &&
               entry("cuOccupancyMaxActiveBlocksPerMultiprocessor", x.OccupancyMaxActiveBlocksPerMultiprocessor) &&
               entry("cuLaunchKernel", x.LaunchKernel) && entry("cuLaunchCooperativeKernel", x.LaunchCooperativeKernel);
        return x;
    }();
    return d;
}

// NVRTC, opened at first use (libnvrtc.so.12 of the CUDA toolkit or of the
// Python environment's nvidia-cuda-nvrtc wheel): not a link dependency.
struct Nvrtc {
    nvrtcResult (*CreateProgram)(nvrtcProgram *, const char *, const char *, int, const char *const *,
                                 const char *const *) = nullptr;
    nvrtcResult (*DestroyProgram)(nvrtcProgram *) = nullptr;
    nvrtcResult (*AddNameExpression)(nvrtcProgram, const char *) = nullptr;
    nvrtcResult (*CompileProgram)(nvrtcProgram, int, const char *const *) = nullptr;
    nvrtcResult (*GetProgramLogSize)(nvrtcProgram, size_t *) = nullptr;
    nvrtcResult (*GetProgramLog)(nvrtcProgram, char *) = nullptr;
    nvrtcResult (*GetLoweredName)(nvrtcProgram, const char *, const char **) = nullptr;
    nvrtcResult (*GetCUBINSize)(nvrtcProgram, size_t *) = nullptr;
    nvrtcResult (*GetCUBIN)(nvrtcProgram, char *) = nullptr;
    bool ok = false;
};

template <class F>
bool sym(void *h, const char *name, F &f) {
    f = reinterpret_cast<F>(dlsym(h, name));
    return f != nullptr;
}

const Nvrtc &nvrtc() {
    static Nvrtc n = [] {
        Nvrtc x;
        void *h = nullptr;
        for (const char *path : {"libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so"})
            if ((h = dlopen(path, RTLD_NOW | RTLD_LOCAL))) break;
        if (!h) return x;
        x.ok = sym(h, "nvrtcCreateProgram", x.CreateProgram) && sym(h, "nvrtcDestroyProgram", x.DestroyProgram) &&
               sym(h, "nvrtcAddNameExpression", x.AddNameExpression) &&
               sym(h, "nvrtcCompileProgram", x.CompileProgram) &&
               sym(h, "nvrtcGetProgramLogSize", x.GetProgramLogSize) && sym(h, "nvrtcGetProgramLog", x.GetProgramLog) &&
               sym(h, "nvrtcGetLoweredName", x.GetLoweredName) && sym(h, "nvrtcGetCUBINSize", x.GetCUBINSize) &&
               sym(h, "nvrtcGetCUBIN", x.GetCUBIN);
        return x;
    }();
    return n;
}

std::string cu_err(CUresult r) {
    const char *s = nullptr;
    if (drv().GetErrorString) drv().GetErrorString(r, &s);
    return s ? s : "CUDA driver error " + std::to_string((int)r);
}

}  // namespace

tm_status rtc_kernel(uint64_t code, bool gen, int mode, RtcKernel *out) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaFree(nullptr) != cudaSuccess)   // primary context current
        return fail(TM_ECUDA, "no CUDA device for tm_motif_specialise");
    if (!drv().ok) return fail(TM_ECUDA, "CUDA driver entry points unavailable");
    const Nvrtc &R = nvrtc();
    if (!R.ok) return fail(TM_ECUDA, "libnvrtc.so.12 not found (runtime specialisation needs NVRTC)");
    const auto key = std::make_tuple(dev, code, gen, mode);
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_cache.find(key);
    if (it == g_cache.end()) {
        const std::string plan = "tmg::PlanC<" + std::to_string(code) + "ull, " + (gen ? "true" : "false") + ">";
        const std::string src = "#include \"mine.cuh\"\n"
                                "extern \"C\" __device__ int tm_rtc_smem_words = tmg::Layout<" + plan + ", " +
                                std::to_string(mode) + ">::warp_words();\n";
        const std::string expr = "&tmg::mine_kernel<" + plan + ", " + std::to_string(mode) + ">";
        const char *hdr[3] = {kRtcInternal, kRtcMine, kRtcApiMacros};
        const char *hname[3] = {"tm_internal.cuh", "mine.cuh", "../../include/tmotif.h"};
        nvrtcProgram prog;
        if (R.CreateProgram(&prog, src.c_str(), "tm_rtc.cu", 3, hdr, hname) != NVRTC_SUCCESS)
            return fail(TM_ECUDA, "nvrtcCreateProgram failed");
        struct ProgFree { nvrtcProgram *p; ~ProgFree() { nvrtc().DestroyProgram(p); } } pf{&prog};
        R.AddNameExpression(prog, expr.c_str());
        int major = 0, minor = 0;
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
        const std::string arch = "-arch=sm_" + std::to_string(major * 10 + minor) + "a";
        const char *opts[] = {arch.c_str(), "-std=c++17", "-default-device", "-lineinfo"};
        if (R.CompileProgram(prog, 4, opts) != NVRTC_SUCCESS) {
            size_t n = 0;
            R.GetProgramLogSize(prog, &n);
            std::string log(n, '\0');
            R.GetProgramLog(prog, &log[0]);
            return fail(TM_ECUDA, "NVRTC compile of " + expr + " failed:\n" + log);
        }
        const char *lowered = nullptr;
        R.GetLoweredName(prog, expr.c_str(), &lowered);
        size_t nc = 0;
        R.GetCUBINSize(prog, &nc);
        std::vector<char> cubin(nc);
        R.GetCUBIN(prog, cubin.data());
        Entry e;
        CUresult r = drv().ModuleLoadData(&e.mod, cubin.data());
        if (r == CUDA_SUCCESS) r = drv().ModuleGetFunction(&e.fn, e.mod, lowered);
        CUdeviceptr g = 0;
        size_t gb = 0;
        if (r == CUDA_SUCCESS) r = drv().ModuleGetGlobal(&g, &gb, e.mod, "tm_rtc_smem_words");
        int words = 0;
        if (r == CUDA_SUCCESS) r = drv().MemcpyDtoH(&words, g, sizeof words);
        if (r != CUDA_SUCCESS) return fail(TM_ECUDA, "loading the specialised kernel: " + cu_err(r));
        e.smem_per_warp = words * (int)sizeof(uint32_t);
        it = g_cache.emplace(key, e).first;
    }
    out->fn = it->second.fn;
    out->smem_per_warp = it->second.smem_per_warp;
    return TM_OK;
}

cudaError_t rtc_set_smem(void *fn, int bytes) {
    const CUresult r = drv().FuncSetAttribute((CUfunction)fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, bytes);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t rtc_occupancy(void *fn, int threads, size_t smem, int *per_sm) {
    const CUresult r = drv().OccupancyMaxActiveBlocksPerMultiprocessor(per_sm, (CUfunction)fn, threads, smem);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t rtc_launch(void *fn, unsigned grid, int threads, size_t smem, cudaStream_t s, const MineParams &p,
                       bool coop) {
    void *args[] = {const_cast<MineParams *>(&p)};
    const CUresult r = coop ? drv().LaunchCooperativeKernel((CUfunction)fn, grid, 1, 1, threads, 1, 1, (unsigned)smem,
                                                            (CUstream)s, args)
                            : drv().LaunchKernel((CUfunction)fn, grid, 1, 1, threads, 1, 1, (unsigned)smem,
                                                 (CUstream)s, args, nullptr);
    if (r == CUDA_ERROR_COOPERATIVE_LAUNCH_TOO_LARGE) return cudaErrorCooperativeLaunchTooLarge;
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorLaunchFailure;
}

}  // namespace tmg
