// NVRTC compilation of emitted assembly kernels for sm_100a (the runtime
// compilation step of the paper, §5; the reference only renders the
// template text, kernel.cpp:409-449, and never compiles it -- SPEC.md:15).
#include <dlfcn.h>
#include <nvrtc.h>

#include <chrono>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <mutex>
#include <regex>
#include <sstream>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "femforge_b200.h"
#include "runtime.hpp"

namespace ffb {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(FF_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

namespace {

// NVRTC of this CUDA toolkit, loaded privately (RTLD_LOCAL, by full path):
// a host process (e.g. PyTorch) may already have loaded another NVRTC with the
// same SONAME, which would otherwise win symbol resolution and compile with
// an older PTX ISA (no 256-bit loads, different sm_100a code generation).
struct Nvrtc {
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  decltype(&nvrtcGetErrorString) error = nullptr;
  decltype(&nvrtcVersion) version = nullptr;
  std::string path;
};

const Nvrtc& nvrtc() {
  static const Nvrtc api = [] {
    Nvrtc a;
    std::vector<std::string> candidates;
    for (const char* env : {"FF_NVRTC", "CUDA_HOME", "CUDA_PATH"})
      if (const char* v = std::getenv(env)) {
        const std::string d(v);
        candidates.push_back(std::string(env) == "FF_NVRTC" ? d : d + "/lib64/libnvrtc.so.12");
      }
    candidates.push_back("/usr/local/cuda/lib64/libnvrtc.so.12");
    candidates.push_back("libnvrtc.so.12");
    void* h = nullptr;
    for (const std::string& c : candidates)
      if ((h = dlopen(c.c_str(), RTLD_NOW | RTLD_LOCAL))) {
        a.path = c;
        break;
      }
    if (!h) throw Error(FF_E_NVRTC, "cannot load libnvrtc.so.12 (set FF_NVRTC or CUDA_HOME)");
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) throw Error(FF_E_NVRTC, std::string("libnvrtc: missing ") + name);
    };
    sym(a.create, "nvrtcCreateProgram");
    sym(a.compile, "nvrtcCompileProgram");
    sym(a.log_size, "nvrtcGetProgramLogSize");
    sym(a.log, "nvrtcGetProgramLog");
    sym(a.cubin_size, "nvrtcGetCUBINSize");
    sym(a.cubin, "nvrtcGetCUBIN");
    sym(a.destroy, "nvrtcDestroyProgram");
    sym(a.error, "nvrtcGetErrorString");
    sym(a.version, "nvrtcVersion");
    return a;
  }();
  return api;
}

const char* const kOptions[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "--diag-suppress=177",
                                "--ptxas-options=-v"};

std::mutex g_cache_mu;
std::unordered_map<std::string, CompiledModule> g_cache;

std::string cache_key(const std::string& src) {
  int major = 0, minor = 0;
  nvrtc().version(&major, &minor);
  std::string k = src + "\nnvrtc " + std::to_string(major) + "." + std::to_string(minor);
  for (const char* o : kOptions) k += '\n', k += o;
  return k;
}

std::string disk_path(const std::string& key) {
  const char* dir = std::getenv("FF_CUBIN_CACHE");
  if (!dir || !*dir) return {};
  std::ostringstream os;
  os << dir << "/ff_" << std::hex << std::hash<std::string>()(key) << "_" << key.size() << ".cubin";
  return os.str();
}

// ptxas -v lines of the element kernel (ff_assemble_atomic; else the first
// entry function of the module)
void parse_resources(CompiledModule& m) {
  const std::regex entry("entry function '([A-Za-z_0-9]+)'");
  std::string block = m.log;
  for (auto it = std::sregex_iterator(m.log.begin(), m.log.end(), entry); it != std::sregex_iterator(); ++it) {
    if ((*it)[1] != "ff_assemble_atomic") continue;
    const std::size_t at = static_cast<std::size_t>(it->position());
    const std::size_t next = m.log.find("entry function", at + 1);
    block = m.log.substr(at, next == std::string::npos ? std::string::npos : next - at);
    break;
  }
  std::smatch r;
  if (std::regex_search(block, r, std::regex("Used ([0-9]+) registers"))) m.registers = std::stoi(r[1]);
  if (std::regex_search(block, r, std::regex("([0-9]+) bytes smem"))) m.shared_bytes = std::stoi(r[1]);
}

}  // namespace

CompiledModule nvrtc_compile(const std::string& source, const std::string& name) {
  const std::string key = cache_key(source);
  {
    std::lock_guard<std::mutex> g(g_cache_mu);
    auto it = g_cache.find(key);
    if (it != g_cache.end()) return it->second;
  }
  CompiledModule m;
  const std::string path = disk_path(key);
  if (!path.empty()) {
    std::ifstream in(path, std::ios::binary);
    if (in) {
      std::stringstream ss;
      ss << in.rdbuf();
      std::string blob = ss.str();
      const std::size_t cut = blob.find('\0');
      if (cut != std::string::npos && cut + 1 < blob.size()) {
        m.log = blob.substr(0, cut);
        m.cubin = blob.substr(cut + 1);
        parse_resources(m);
        std::lock_guard<std::mutex> g(g_cache_mu);
        g_cache.emplace(key, m);
        return m;
      }
    }
  }
  const auto t0 = std::chrono::steady_clock::now();
  const Nvrtc& api = nvrtc();
  nvrtcProgram prog = nullptr;
  if (api.create(&prog, source.c_str(), name.c_str(), 0, nullptr, nullptr) != NVRTC_SUCCESS)
    throw Error(FF_E_NVRTC, "nvrtcCreateProgram failed");
  const nvrtcResult rc = api.compile(prog, static_cast<int>(sizeof kOptions / sizeof kOptions[0]), kOptions);
  std::size_t log_size = 0;
  api.log_size(prog, &log_size);
  m.log.assign(log_size, '\0');
  if (log_size) api.log(prog, m.log.data());
  while (!m.log.empty() && m.log.back() == '\0') m.log.pop_back();
  if (rc != NVRTC_SUCCESS) {
    api.destroy(&prog);
    throw Error(FF_E_NVRTC, std::string("NVRTC compilation failed (") + api.error(rc) + "):\n" + m.log);
  }
  std::size_t n = 0;
  api.cubin_size(prog, &n);
  m.cubin.assign(n, '\0');
  api.cubin(prog, m.cubin.data());
  api.destroy(&prog);
  m.ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  parse_resources(m);
  if (!path.empty()) {
    std::ofstream out(path, std::ios::binary);
    out << m.log << '\0' << m.cubin;
  }
  std::lock_guard<std::mutex> g(g_cache_mu);
  g_cache.emplace(key, m);
  return m;
}

}  // namespace ffb
