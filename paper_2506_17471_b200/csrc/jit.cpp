// jit.cpp — NVRTC compilation of emitted kernels for sm_100a, cached by source
// hash in memory and on disk ($FEMGPU_CACHE, default ~/.cache/femgpu), loaded
// with the CUDA runtime library API (cudaLibraryLoadData / cudaLibraryGetKernel),
// so libfemgpu needs no libcuda link dependency and loads on GPU-less hosts.
#include <nvrtc.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <sys/stat.h>
#include <unistd.h>

#include "femgpu_internal.hpp"

namespace femgpu {

namespace {

uint64_t fnv1a(const std::string& s, uint64_t h = 0xcbf29ce484222325ULL) {
    for (unsigned char c : s) {
        h ^= c;
        h *= 0x100000001b3ULL;
    }
    return h;
}

std::string cache_dir() {
    if (const char* e = std::getenv("FEMGPU_CACHE")) return e;
    const char* home = std::getenv("HOME");
    return std::string(home ? home : "/tmp") + "/.cache/femgpu";
}

void mkdirs(const std::string& path) {
    std::string cur;
    std::stringstream ss(path);
    std::string part;
    if (!path.empty() && path[0] == '/') cur = "/";
    while (std::getline(ss, part, '/')) {
        if (part.empty()) continue;
        cur += part + "/";
        ::mkdir(cur.c_str(), 0755);
    }
}

#define NVRTC_CHECK(x)                                                              \
    do {                                                                            \
        nvrtcResult r_ = (x);                                                       \
        if (r_ != NVRTC_SUCCESS) fail(FEMGPU_E_JIT, std::string(#x) + ": " + nvrtcGetErrorString(r_)); \
    } while (0)

std::mutex g_jit_mu;
std::map<std::string, std::shared_ptr<Module>> g_modules;  // key: device|source hash

}  // namespace

std::vector<char> jit_compile(const std::string& source, bool strict, std::string* log_out) {
    int major = 0, minor = 0;
    nvrtcVersion(&major, &minor);
    const std::string opts_key = std::string(strict ? "strict" : "fast") + "/nvrtc" + std::to_string(major) + "." +
                                 std::to_string(minor) + "/sm_100a/v3";
    const uint64_t h = fnv1a(source, fnv1a(opts_key));
    char hex[32];
    std::snprintf(hex, sizeof hex, "%016llx", static_cast<unsigned long long>(h));
    const std::string dir = cache_dir();
    const std::string path = dir + "/" + hex + ".cubin";
    {
        std::ifstream in(path, std::ios::binary);
        if (in) {
            std::vector<char> bin((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
            if (!bin.empty()) return bin;
        }
    }
    nvrtcProgram prog;
    NVRTC_CHECK(nvrtcCreateProgram(&prog, source.c_str(), "femgpu_kernel.cu", 0, nullptr, nullptr));
    std::vector<const char*> opts = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo",
                                     strict ? "--fmad=false" : "--fmad=true", "-DNDEBUG"};
    const nvrtcResult rc = nvrtcCompileProgram(prog, static_cast<int>(opts.size()), opts.data());
    size_t log_size = 0;
    nvrtcGetProgramLogSize(prog, &log_size);
    std::string log(log_size, '\0');
    if (log_size) nvrtcGetProgramLog(prog, log.data());
    if (log_out) *log_out = log;
    if (rc != NVRTC_SUCCESS) {
        nvrtcDestroyProgram(&prog);
        fail(FEMGPU_E_JIT, std::string("nvrtc compile failed: ") + nvrtcGetErrorString(rc) + "\n" + log);
    }
    size_t n = 0;
    NVRTC_CHECK(nvrtcGetCUBINSize(prog, &n));
    std::vector<char> bin(n);
    NVRTC_CHECK(nvrtcGetCUBIN(prog, bin.data()));
    nvrtcDestroyProgram(&prog);
    try {
        mkdirs(dir);
        // per-process temporary + rename: concurrent ranks compiling the same kernel never see a torn file
        const std::string tmp = path + ".tmp" + std::to_string(static_cast<long long>(::getpid()));
        std::ofstream out(tmp, std::ios::binary);
        out.write(bin.data(), static_cast<std::streamsize>(bin.size()));
        out.close();
        std::rename(tmp.c_str(), path.c_str());
    } catch (...) {
    }
    return bin;
}

std::shared_ptr<Module> get_module(const Signature& sig, const KernelPlan& kp) {
    EmitResult em = emit_kernel(sig, kp);
    int dev = 0;
    FG_CUDA(cudaGetDevice(&dev));
    const std::string key = std::to_string(dev) + "|" + std::to_string(kp.strict) + "|" +
                            std::to_string(fnv1a(em.source));
    {
        std::lock_guard<std::mutex> lk(g_jit_mu);
        auto it = g_modules.find(key);
        if (it != g_modules.end()) return it->second;
    }
    // NVRTC outside the lock: the automatic schedule compiles its candidates from several threads
    std::string log;
    std::vector<char> bin = jit_compile(em.source, kp.strict, &log);
    std::lock_guard<std::mutex> lk(g_jit_mu);
    auto it = g_modules.find(key);
    if (it != g_modules.end()) return it->second;  // another thread compiled it meanwhile
    auto m = std::make_shared<Module>();
    FG_CUDA(cudaLibraryLoadData(&m->lib, bin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
    FG_CUDA(cudaLibraryGetKernel(&m->fast, m->lib, em.kernel.c_str()));
    FG_CUDA(cudaLibraryGetKernel(&m->checked, m->lib, em.kernel_checked.c_str()));
    if (em.smem_bytes > 48 * 1024 && em.smem_bytes <= 227 * 1024) {
        FG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(m->fast),
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(em.smem_bytes)));
        FG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(m->checked),
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(em.smem_bytes)));
    }
    {
        int occ = 0, dev_sms = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, reinterpret_cast<const void*>(m->fast), kp.block,
                                                          em.smem_bytes) == cudaSuccess && occ > 0)
            m->occupancy = occ;
        else
            m->occupancy = std::max(1, kp.min_blocks);
        cudaGetLastError();
        if (cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && dev_sms > 0)
            m->sms = dev_sms;
    }
    cudaFuncAttributes attr{};
    if (cudaFuncGetAttributes(&attr, reinterpret_cast<const void*>(m->fast)) == cudaSuccess) {
        m->regs = attr.numRegs;
        m->local_bytes = static_cast<long long>(attr.localSizeBytes);  // > 0: register spills to local memory
    }
    cudaGetLastError();
    m->emitted = std::move(em);
    g_modules[key] = m;
    return m;
}

}  // namespace femgpu
