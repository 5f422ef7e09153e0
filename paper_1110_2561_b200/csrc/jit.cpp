// Per-lattice specialisation of the hoisted kernel with NVRTC.
//
// k1_body.cuh is compiled a second time at run time with every lattice
// constant (masks, shifts, the 128-entry copy offset table, layout strides,
// loop width) turned into a constexpr, for sm_100a.  The copy offsets then
// fold into the shared RED's address immediate and the per-group masks into
// LOP3 immediates, which removes the uniform-register loads the ahead-of-time
// kernel needs.  NVRTC is loaded with dlopen; if it is
// missing or a compile fails the caller falls back to the ahead-of-time
// kernel (same arithmetic, same results) and isd_kernel_info() says so.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <future>
#include <map>
#include <mutex>
#include <thread>
#include <sstream>
#include <string>
#include <vector>

#include "isd_internal.h"

namespace isd {

static const char kBodySource[] =
#include "k1_body_str.inc"
    ;

// ---- minimal NVRTC binding -------------------------------------------------
typedef int nvrtcResult_t;
typedef struct _nvrtcProgram* nvrtcProgram_t;
struct Nvrtc {
  bool ok = false;
  std::string why;
  nvrtcResult_t (*create)(nvrtcProgram_t*, const char*, const char*, int,
                          const char* const*, const char* const*) = nullptr;
  nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char* const*) = nullptr;
  nvrtcResult_t (*cubin_size)(nvrtcProgram_t, size_t*) = nullptr;
  nvrtcResult_t (*cubin)(nvrtcProgram_t, char*) = nullptr;
  nvrtcResult_t (*log_size)(nvrtcProgram_t, size_t*) = nullptr;
  nvrtcResult_t (*log)(nvrtcProgram_t, char*) = nullptr;
  nvrtcResult_t (*destroy)(nvrtcProgram_t*) = nullptr;
};

static Nvrtc& nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    for (const char* name : {"libnvrtc.so.12", "libnvrtc.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
      if (h) break;
    }
    if (!h) {
      n.why = "libnvrtc not found";
      return;
    }
    n.create = (decltype(n.create))dlsym(h, "nvrtcCreateProgram");
    n.compile = (decltype(n.compile))dlsym(h, "nvrtcCompileProgram");
    n.cubin_size = (decltype(n.cubin_size))dlsym(h, "nvrtcGetCUBINSize");
    n.cubin = (decltype(n.cubin))dlsym(h, "nvrtcGetCUBIN");
    n.log_size = (decltype(n.log_size))dlsym(h, "nvrtcGetProgramLogSize");
    n.log = (decltype(n.log))dlsym(h, "nvrtcGetProgramLog");
    n.destroy = (decltype(n.destroy))dlsym(h, "nvrtcDestroyProgram");
    n.ok = n.create && n.compile && n.cubin_size && n.cubin && n.log_size &&
           n.log && n.destroy;
    if (!n.ok) n.why = "libnvrtc lacks a required symbol";
  });
  return n;
}

// ---- source generation -----------------------------------------------------
template <typename V>
static void emit_switch(std::ostringstream& o, const char* type,
                        const char* name, const V* vals, int n,
                        const char* suffix) {
  o << "  __device__ __forceinline__ static constexpr " << type << " "
    << name << "(int i) {\n    switch (i) {\n";
  for (int i = 0; i < n; ++i)
    o << "      case " << i << ": return " << vals[i] << suffix << ";\n";
  o << "    }\n    return 0;\n  }\n";
}

static std::string generate(const HoistParams& P, int nc, bool dbl,
                            bool debug_bounds) {
  std::ostringstream o;
  o << "typedef unsigned int uint32_t;\n"
       "typedef unsigned long long uint64_t;\n"
       "typedef int int32_t;\n";
  if (knob_long("ISD_PROBE", 0)) o << "#define ISD_PROBE 1\n";
  if (debug_bounds)
    o << "#define ISD_CHECK_ADDR(a, lo, bytes) do { if ((unsigned)((a) - "
         "(lo)) >= (bytes) || ((a) & 3u)) __trap(); } while (0)\n";
  o << kBodySource << "\n";
  o << "struct JitTraits {\n";
  auto c32 = [&](const char* name, unsigned long long v) {
    o << "  __device__ __forceinline__ static constexpr uint32_t " << name
      << "() { return " << v << "u; }\n";
  };
  auto c64 = [&](const char* name, unsigned long long v) {
    o << "  __device__ __forceinline__ static constexpr uint64_t " << name
      << "() { return " << v << "ull; }\n";
  };
  c32("k", P.k);
  c32("nloop", 1u << P.l);
  c64("above_k", P.above_k);
  c64("odd_mask", P.odd_mask);
  c32("loop_mask", P.loop_mask);
  c32("e_parity", P.e_parity);
  c32("e_mode", P.e_mode);
  c32("row_bytes", P.row_bytes);
  c32("e_bytes", P.e_bytes);
  o << "  __device__ __forceinline__ static constexpr int32_t plane_bytes() "
       "{ return "
    << P.plane_bytes << "; }\n";
  c32("row_words", P.row_words);
  c32("e_words", P.e_words);
  c32("plane_words", P.plane_words);
  c32("stride", P.stride);
  c32("nbins", P.nbins);
  c32("hist_words", P.hist_words);
  c32("n_hist", P.n_hist);
  emit_switch(o, "uint32_t", "shift", P.shift, nc, "u");
  emit_switch(o, "uint64_t", "mask", P.mask, nc, "ull");
  emit_switch(o, "uint64_t", "jneg", P.jneg, nc, "ull");
  emit_switch(o, "uint32_t", "mvar", P.mvar, nc, "u");
  emit_switch(o, "uint64_t", "nm1", P.nm1, kCopyBits, "ull");
  emit_switch(o, "uint64_t", "jn1", P.jn1, kCopyBits, "ull");
  emit_switch(o, "uint64_t", "nm2", P.nm2, kCopyBits, "ull");
  emit_switch(o, "uint64_t", "jn2", P.jn2, kCopyBits, "ull");
  emit_switch(o, "uint32_t", "nm1v", P.nm1v, kCopyBits, "u");
  emit_switch(o, "uint32_t", "jn1v", P.jn1v, kCopyBits, "u");
  emit_switch(o, "uint32_t", "nm2v", P.nm2v, kCopyBits, "u");
  emit_switch(o, "uint32_t", "jn2v", P.jn2v, kCopyBits, "u");
  emit_switch(o, "int32_t", "degree", P.degree, kCopyBits, "");
  uint32_t koff[kCopies];
  for (int c = 0; c < kCopies; ++c) koff[c] = (uint32_t)P.koff[c];
  emit_switch(o, "uint32_t", "koff", koff, kCopies, "u");
  emit_switch(o, "uint32_t", "pair_bytes", P.pair_bytes, 2, "u");
  emit_switch(o, "uint32_t", "pair_words", P.pair_words, 2, "u");
  emit_switch(o, "int32_t", "pair_deg", P.pair_deg, 2, "");
  o << "  __device__ __forceinline__ static constexpr int32_t pair_both() "
       "{ return "
    << P.pair_both << "; }\n";
  c32("band_rows", P.band_rows);
  // Gray sites
  o << "  __host__ __device__ static constexpr int gray() { return " << P.gray
    << "; }\n";
  // mode 3: the cluster's external degree as a compile-time constant (the
  // two-stage flush sizes register arrays with it)
  o << "  __host__ __device__ static constexpr int tri_r() { return "
    << (P.pair == 3 ? (int)P.pair_deg[0] : -1) << "; }\n";
  c32("g_mask", P.g_mask);
  emit_switch(o, "uint32_t", "g_bit", P.g_bit, kMaxGray, "u");
  emit_switch(o, "uint64_t", "g_nm1", P.g_nm1, kMaxGray, "ull");
  emit_switch(o, "uint64_t", "g_jn1", P.g_jn1, kMaxGray, "ull");
  emit_switch(o, "uint64_t", "g_nm2", P.g_nm2, kMaxGray, "ull");
  emit_switch(o, "uint64_t", "g_jn2", P.g_jn2, kMaxGray, "ull");
  emit_switch(o, "uint32_t", "g_nm1v", P.g_nm1v, kMaxGray, "u");
  emit_switch(o, "uint32_t", "g_jn1v", P.g_jn1v, kMaxGray, "u");
  emit_switch(o, "uint32_t", "g_nm2v", P.g_nm2v, kMaxGray, "u");
  emit_switch(o, "uint32_t", "g_jn2v", P.g_jn2v, kMaxGray, "u");
  emit_switch(o, "int32_t", "g_deg", P.g_deg, kMaxGray, "");
  emit_switch(o, "int32_t", "g_csum", P.g_csum, kMaxGray, "");
  emit_switch(o, "int32_t", "g_odd", P.g_odd, kMaxGray, "");
  o << "  __device__ __forceinline__ static constexpr int32_t g_cdelta(int g, "
       "int q) {\n";
  for (int g = 0; g < kMaxGray; ++g)
    for (int q = 0; q < kCopyBits; ++q)
      o << "    if (g == " << g << " && q == " << q << ") return "
        << P.g_cdelta[g][q] << ";\n";
  o << "    return 0;\n  }\n";
  o << "};\n";
  o << "extern \"C\" __global__ void __launch_bounds__("
    << (P.pair >= 2 ? kWideThreads : kThreads)
    << ") k1_jit(unsigned long long run_begin, unsigned long long nruns,\n"
       "    unsigned long long hi_step, unsigned long long lane_mask,\n"
       "    const IsdLanes lanes, const IsdBandItem* items,\n"
       "    unsigned int n_items, int free_bits, unsigned int* claim,\n"
       "    const IsdSlotMap smap, unsigned long long* item_clk,\n"
       "    unsigned long long* __restrict__ out) {\n"
       "  extern __shared__ __align__(16) unsigned int hist[];\n"
       "  const JitTraits L;\n"
       "  k1_hoisted_body<"
    << nc << ", " << (dbl ? "true" : "false") << ", "
    << P.pair << ">(L, run_begin, nruns, hi_step, lane_mask, lanes, items,\n"
       "      n_items, free_bits, claim, smap, item_clk, hist, out);\n}\n";
  return o.str();
}

// ---- cache -----------------------------------------------------------------
// Two levels, both filled without holding a lock across a compile (so the
// host threads of different GPUs, and the autotuner's finalists, compile in
// parallel): cubins by generated source (memory, then the disk cache of
// cache.cpp), and loaded kernels by (source, device).
struct JitKernel {
  bool ok = false;
  std::string why;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
  int per_sm = 0;  // resident blocks per SM (grid = per_sm x SMs)
  int threads = kThreads;
};

struct Cubin {
  bool ok = false;
  std::string why;
  std::string bytes;
};

static std::mutex g_jit_mu;
static std::map<std::string, std::shared_future<Cubin>> g_cubins;
static std::map<std::string, std::shared_future<JitKernel>> g_jit;

// (-default-device: the body's generic lambdas carry no execution-space
// annotation, which NVRTC would otherwise read as host functions)
static const char* const kNvrtcOpts[] = {"--gpu-architecture=sm_100a",
                                         "-std=c++17", "-lineinfo",
                                         "-default-device"};

// The specialised kernel's source (it holds every lattice constant, so it
// identifies the kernel).
static std::string jit_source(const HoistParams& P) {
#ifdef ISD_DEBUG_BOUNDS
  const bool debug_bounds = true;
#else
  const bool debug_bounds = false;
#endif
  return generate(P, (int)P.n_classes, P.has_double != 0, debug_bounds);
}

// NVRTC compile of one source (host only).
static Cubin compile_source(const std::string& src) {
  NvtxRange nvtx("isd:nvrtc compile");
  Cubin out;
  Nvrtc& nv = nvrtc();
  if (!nv.ok) {
    out.why = nv.why;
    return out;
  }
  nvrtcProgram_t prog = nullptr;
  if (nv.create(&prog, src.c_str(), "k1_jit.cu", 0, nullptr, nullptr) != 0) {
    out.why = "nvrtcCreateProgram failed";
    return out;
  }
  const int rc = nv.compile(
      prog, (int)(sizeof kNvrtcOpts / sizeof kNvrtcOpts[0]), kNvrtcOpts);
  if (rc != 0) {
    size_t n = 0;
    nv.log_size(prog, &n);
    std::string log(n, '\0');
    if (n) nv.log(prog, &log[0]);
    out.why = "NVRTC compile failed: " + log.substr(0, 600);
    nv.destroy(&prog);
    return out;
  }
  size_t n = 0;
  nv.cubin_size(prog, &n);
  out.bytes.resize(n);
  nv.cubin(prog, &out.bytes[0]);
  nv.destroy(&prog);
  out.ok = true;
  return out;
}

// The cubin of P's kernel: memoised per process, then the disk cache, then
// NVRTC.  Concurrent callers of one source share a single compile.
static Cubin get_cubin(const HoistParams& P) {
  const std::string src = jit_source(P);
  std::string key = src;
  for (const char* o : kNvrtcOpts) key += std::string("|") + o;
  std::shared_future<Cubin> fut;
  std::promise<Cubin> prom;
  bool mine = false;
  {
    std::lock_guard<std::mutex> lock(g_jit_mu);
    auto it = g_cubins.find(key);
    if (it == g_cubins.end()) {
      fut = prom.get_future().share();
      g_cubins.emplace(key, fut);
      mine = true;
    } else {
      fut = it->second;
    }
  }
  if (mine) {
    Cubin c;
    if (cache_get("cubin", key, &c.bytes) && !c.bytes.empty()) {
      c.ok = true;
    } else {
      c = compile_source(src);
      if (c.ok) cache_put("cubin", key, c.bytes);
    }
    prom.set_value(std::move(c));
  }
  Cubin c = fut.get();
  // inspection knob: ISD_JIT_DUMP=<path> writes the cubin (cuobjdump -sass)
  std::string dump;
  if (c.ok && knob_str("ISD_JIT_DUMP", &dump) && !dump.empty()) {
    if (FILE* f = std::fopen(dump.c_str(), "wb")) {
      std::fwrite(c.bytes.data(), 1, c.bytes.size(), f);
      std::fclose(f);
    }
  }
  return c;
}

int jit_compile_check(const HoistParams& P, std::string* why) {
  const std::string src = jit_source(P);
  Cubin c = compile_source(src);
  if (!c.ok) {
    *why = c.why;
    return 0;
  }
  std::string dump;  // (ISD_JIT_DUMP: inspect the SASS without a GPU)
  if (knob_str("ISD_JIT_DUMP", &dump) && !dump.empty()) {
    if (FILE* f = std::fopen(dump.c_str(), "wb")) {
      std::fwrite(c.bytes.data(), 1, c.bytes.size(), f);
      std::fclose(f);
    }
  }
  return (int)c.bytes.size();
}

// Compile (or fetch) the cubins of several kernels concurrently: the
// autotuner's finalists are known before any of them is timed.
void jit_prefetch(const std::vector<HoistParams>& ps) {
  if (!nvrtc().ok || ps.empty()) return;
  std::vector<std::thread> pool;
  for (const HoistParams& p : ps) pool.emplace_back([p] { get_cubin(p); });
  for (std::thread& t : pool) t.join();
}

// The caller's stream may be capturing a graph: loading (and probing) a
// module is not part of the captured work, so this thread steps out of the
// capture rules while it builds a kernel.
struct RelaxedCapture {
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  RelaxedCapture() { cudaThreadExchangeStreamCaptureMode(&mode); }
  ~RelaxedCapture() { cudaThreadExchangeStreamCaptureMode(&mode); }
};

static JitKernel build_kernel(const HoistParams& P0) {
  JitKernel jk;
  RelaxedCapture relaxed;
  // A Gray walk over many sites is long straight-line code: where it
  // spills more than a few per-run values to local memory (c4 at five
  // sites: 80 B of stack; at four: 48 B, and 1.084 -> 1.065 ms), one site
  // fewer is faster — step down until the stack is small (c5's 24 B are
  // two values saved once per run of 512 REDs).
  constexpr size_t kSpillBytesOk = 64;
  HoistParams P = P0;
  for (;;) {
    Cubin probe = get_cubin(P);
    if (!probe.ok || P.gray <= 2) break;
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kern = nullptr;
    cudaFuncAttributes attr;
    std::memset(&attr, 0, sizeof attr);
    cudaError_t pe = cudaLibraryLoadData(&lib, probe.bytes.data(), nullptr,
                                         nullptr, 0, nullptr, nullptr, 0);
    if (pe == cudaSuccess) pe = cudaLibraryGetKernel(&kern, lib, "k1_jit");
    if (pe == cudaSuccess) pe = cudaFuncGetAttributes(&attr, (const void*)kern);
    if (lib) cudaLibraryUnload(lib);
    if (pe != cudaSuccess) {
      cudaGetLastError();
      break;
    }
    if (attr.localSizeBytes <= kSpillBytesOk) break;
    P.gray -= 1;
    P.g_mask &= ~P.g_bit[P.gray];
  }
  Cubin cubin = get_cubin(P);
  if (!cubin.ok) {
    jk.why = cubin.why;
    return jk;
  }
  cudaError_t e = cudaLibraryLoadData(&jk.lib, cubin.bytes.data(), nullptr,
                                      nullptr, 0, nullptr, nullptr, 0);
  if (e == cudaSuccess) e = cudaLibraryGetKernel(&jk.kern, jk.lib, "k1_jit");
  const size_t smem = (size_t)P.n_hist * P.hist_words * 4;
  if (e != cudaSuccess) {
    jk.why = std::string("loading the JIT kernel: ") + cudaGetErrorString(e);
    cudaGetLastError();
    return jk;
  }
  jk.threads = hoisted_block((const void*)jk.kern, smem, 1, P.pair >= 2,
                             &jk.per_sm, P.band_rows > 0);
  jk.ok = true;
  return jk;
}

// Bytes of HoistParams that define the kernel (everything but the launch
// arguments), plus the device: the key of a loaded kernel.
static std::string jit_key(const HoistParams& P, int device) {
  HoistParams q = P;
  q.run_begin = q.run_end = 0;
  q.hi_step = 0;
  q.lane_mask = 0;
  for (int i = 0; i < 5; ++i) q.lane_vec[i] = 0;
  q.band_free_bits = q.band_n_items = 0;  // launch arguments, not constants
  q.band_items = 0;
  q.band_claim = 0;
  for (int j = 0; j < 16; ++j) q.slot_mask[j] = q.slot_rot[j] = 0;
  q.band_clk = 0;
  std::string key(reinterpret_cast<const char*>(&q), sizeof q);
  key += std::to_string(device);
  key += knob_long("ISD_PROBE", 0) ? "|probe" : "";
  return key;
}

// The loaded kernel of P on the current device (built once per process).
static JitKernel get_kernel(const HoistParams& P) {
  int dev = 0;
  cudaGetDevice(&dev);
  const std::string key = jit_key(P, dev);
  std::shared_future<JitKernel> fut;
  std::promise<JitKernel> prom;
  bool mine = false;
  {
    std::lock_guard<std::mutex> lock(g_jit_mu);
    auto it = g_jit.find(key);
    if (it == g_jit.end()) {
      fut = prom.get_future().share();
      g_jit.emplace(key, fut);
      mine = true;
    } else {
      fut = it->second;
    }
  }
  if (mine) prom.set_value(build_kernel(P));
  return fut.get();
}

int jit_ready(const HoistParams& P, std::string* why) {
  const JitKernel jk = get_kernel(P);
  if (!jk.ok && why) *why = jk.why;
  return jk.ok ? 1 : 0;
}

// Launch the specialised kernel for P's run range; returns 1 on success,
// 0 if the JIT path is unavailable (caller falls back), <0 on a launch error.
int launch_hoisted_jit(const HoistParams& P, unsigned long long* out,
                       int sm_count, void* stream, std::string* why) {
  const JitKernel jk = get_kernel(P);
  if (!jk.ok) {
    if (why) *why = jk.why;
    return 0;
  }
  unsigned long long run_begin = P.run_begin;
  unsigned long long nruns = P.run_end - P.run_begin;
  unsigned long long hi_step = P.hi_step;
  unsigned long long lane_mask = P.lane_mask;
  struct {
    unsigned long long v[5];
  } lanes;
  for (int i = 0; i < 5; ++i) lanes.v[i] = P.lane_vec[i];
  const void* items = reinterpret_cast<const void*>(P.band_items);
  unsigned int n_items = P.band_n_items;
  int free_bits = (int)P.band_free_bits;
  void* claim = reinterpret_cast<void*>(P.band_claim);
  struct {
    unsigned int mask[16], rot[16];
  } smap;
  for (int j = 0; j < 16; ++j) {
    smap.mask[j] = P.slot_mask[j];
    smap.rot[j] = P.slot_rot[j];
  }
  void* item_clk = reinterpret_cast<void*>(P.band_clk);
  void* args[] = {&run_begin, &nruns,     &hi_step, &lane_mask, &lanes,    &items,
                  &n_items,   &free_bits, &claim,   &smap,      &item_clk, &out};
  int grid = jk.per_sm * sm_count;
  const uint64_t need = (nruns + jk.threads - 1) / jk.threads;
  if (need < (uint64_t)grid) grid = (int)(need ? need : 1);
  const size_t smem = (size_t)P.n_hist * P.hist_words * 4;
  cudaError_t e = cudaLaunchKernel((const void*)jk.kern, dim3(grid),
                                   dim3(jk.threads), args, smem,
                                   (cudaStream_t)stream);
  if (e != cudaSuccess) return -(int)e;
  return 1;
}

}  // namespace isd
