// bode_program.cu -- run-time-compiled solver specialisations.
//
// The reference's plugin surface is open: any ButcherTableau
// (tableau.py:17-83) and any NumPy callable f(t, y) (stepper.py:19-20).
// The persistent integrator is a template over (tableau, functor), so for a
// pair that is not compiled into libbode the facade generates CUDA source
// (the tableau's coefficients as compile-time constants, the callable
// traced into a device functor) and this file compiles the same templates
// for it with NVRTC (sm_100a) -- the kernels are the ones the built-in
// methods run, specialised for the user's problem, with no interpreter or
// CPU fallback anywhere.  The device headers are embedded at build time
// (gen_rtc_headers.py), NVRTC is loaded with dlopen and modules are driven
// through the driver entry points the runtime exposes, so libbode links
// neither libnvrtc nor libcuda.  Compiled cubins are cached on disk by
// content hash.
#include <cuda.h>
#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "bode_program_host.cuh"
#include "bode_rtc_headers.h"

struct bode_program {
  CUmodule mod = nullptr;
  bode_program_desc desc;
  // [mode]: 0 exact, 1 fast
  CUfunction init[2] = {nullptr, nullptr};
  CUfunction solve[2] = {nullptr, nullptr};
  CUfunction solve_pi = nullptr;  // fast mode, I / PI controller
  CUfunction step[2] = {nullptr, nullptr};
  CUfunction joint[2] = {nullptr, nullptr};
  CUfunction rk = nullptr, initial = nullptr;
};

namespace bode {
namespace {

// ------------------------------------------------------------- NVRTC ----
typedef int nvrtcResult_;
struct Nvrtc {
  nvrtcResult_ (*create)(void**, const char*, const char*, int, const char* const*, const char* const*);
  nvrtcResult_ (*compile)(void*, int, const char* const*);
  nvrtcResult_ (*log_size)(void*, size_t*);
  nvrtcResult_ (*log)(void*, char*);
  nvrtcResult_ (*add_name)(void*, const char*);
  nvrtcResult_ (*lowered)(void*, const char*, const char**);
  nvrtcResult_ (*cubin_size)(void*, size_t*);
  nvrtcResult_ (*cubin)(void*, char*);
  nvrtcResult_ (*destroy)(void**);
  nvrtcResult_ (*version)(int*, int*);
  bool ok = false;
  std::string why;
};

const Nvrtc& nvrtc() {
  static Nvrtc N;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"};
    void* h = nullptr;
    for (const char* nm : names)
      if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) {
      N.why = "NVRTC (libnvrtc.so.12) not found";
      return;
    }
    auto sym = [&](const char* s) { return dlsym(h, s); };
    N.create = (decltype(N.create))sym("nvrtcCreateProgram");
    N.compile = (decltype(N.compile))sym("nvrtcCompileProgram");
    N.log_size = (decltype(N.log_size))sym("nvrtcGetProgramLogSize");
    N.log = (decltype(N.log))sym("nvrtcGetProgramLog");
    N.add_name = (decltype(N.add_name))sym("nvrtcAddNameExpression");
    N.lowered = (decltype(N.lowered))sym("nvrtcGetLoweredName");
    N.cubin_size = (decltype(N.cubin_size))sym("nvrtcGetCUBINSize");
    N.cubin = (decltype(N.cubin))sym("nvrtcGetCUBIN");
    N.destroy = (decltype(N.destroy))sym("nvrtcDestroyProgram");
    N.version = (decltype(N.version))sym("nvrtcVersion");
    N.ok = N.create && N.compile && N.log_size && N.log && N.add_name && N.lowered &&
           N.cubin_size && N.cubin && N.destroy && N.version;
    if (!N.ok) N.why = "NVRTC symbols missing";
  });
  return N;
}

// ------------------------------------------------------ driver entries ----
struct Driver {
  CUresult (*load)(CUmodule*, const void*);
  CUresult (*unload)(CUmodule);
  CUresult (*get_function)(CUfunction*, CUmodule, const char*);
  CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                     unsigned, CUstream, void**, void**);
  CUresult (*occupancy)(int*, CUfunction, int, size_t);
  CUresult (*set_attr)(CUfunction, CUfunction_attribute, int);
  bool ok = false;
};

const Driver& driver() {
  static Driver D;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* s) -> void* {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(s, &fn, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        return nullptr;
      return fn;
    };
    D.load = (decltype(D.load))get("cuModuleLoadData");
    D.unload = (decltype(D.unload))get("cuModuleUnload");
    D.get_function = (decltype(D.get_function))get("cuModuleGetFunction");
    D.launch = (decltype(D.launch))get("cuLaunchKernel");
    D.occupancy = (decltype(D.occupancy))get("cuOccupancyMaxActiveBlocksPerMultiprocessor");
    D.set_attr = (decltype(D.set_attr))get("cuFuncSetAttribute");
    D.ok = D.load && D.unload && D.get_function && D.launch && D.occupancy && D.set_attr;
  });
  return D;
}

cudaError_t as_cuda(CUresult r) {
  return r == CUDA_SUCCESS ? cudaSuccess : (r == CUDA_ERROR_INVALID_VALUE ? cudaErrorInvalidValue
                                                                          : cudaErrorLaunchFailure);
}

// ----------------------------------------------------------- cubin cache ----
uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ull) {
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

std::string cache_dir() {
  const char* e = getenv("BODE_JIT_CACHE");
  if (e && *e) return e;
  const char* home = getenv("HOME");
  return std::string(home && *home ? home : "/tmp") + "/.cache/bode_jit";
}

void mkdirs(const std::string& path) {
  std::string cur;
  for (size_t i = 0; i < path.size(); i++) {
    cur += path[i];
    if (path[i] == '/' && cur.size() > 1) mkdir(cur.c_str(), 0755);
  }
  mkdir(path.c_str(), 0755);
}

bool read_file(const std::string& p, std::string& out) {
  FILE* f = fopen(p.c_str(), "rb");
  if (!f) return false;
  std::vector<char> buf(1 << 16);
  out.clear();
  size_t k;
  while ((k = fread(buf.data(), 1, buf.size(), f)) > 0) out.append(buf.data(), k);
  fclose(f);
  return true;
}

void write_file_atomic(const std::string& p, const std::string& data) {
  const std::string tmp = p + ".tmp" + std::to_string(getpid());
  FILE* f = fopen(tmp.c_str(), "wb");
  if (!f) return;
  const bool ok = fwrite(data.data(), 1, data.size(), f) == data.size();
  fclose(f);
  if (ok) rename(tmp.c_str(), p.c_str());
  else unlink(tmp.c_str());
}

// ------------------------------------------------------- instantiations ----
struct Entry {
  std::string expr;  // name expression handed to NVRTC
  CUfunction* slot;
};

std::vector<Entry> entries(bode_program* p) {
  const bode_program_desc& d = p->desc;
  const std::string M = std::to_string(d.method);
  const char* ops[2] = {"bode::ExactOps", "bode::FastOps"};
  auto F = [&](int m) { return std::string("bode::UserDyn<") + ops[m] + ">"; };
  std::vector<Entry> e;
  if (d.kernels & (BODE_PROGRAM_SOLVE | BODE_PROGRAM_STEP))
    for (int m = 0; m < 2; m++)
      e.push_back({"&bode::bode_init_kernel<" + M + ", " + F(m) + ", " + ops[m] + ">", &p->init[m]});
  if (d.kernels & BODE_PROGRAM_SOLVE) {
    for (int m = 0; m < 2; m++)
      e.push_back({"&bode::bode_persistent_kernel<" + M + ", " + F(m) + ", " + ops[m] +
                       ", false, false>", &p->solve[m]});
    e.push_back({"&bode::bode_persistent_kernel<" + M + ", " + F(1) + ", " + ops[1] + ", false, true>",
                 &p->solve_pi});
  }
  if (d.kernels & BODE_PROGRAM_STEP)
    for (int m = 0; m < 2; m++)
      e.push_back({"&bode::bode_step_kernel<" + M + ", " + F(m) + ", " + ops[m] + ">", &p->step[m]});
  if (d.kernels & BODE_PROGRAM_JOINT)
    for (int m = 0; m < 2; m++)
      e.push_back({"&bode::bode_joint_kernel<" + M + ", " + F(m) + ", " + ops[m] + ">", &p->joint[m]});
  if (d.kernels & BODE_PROGRAM_UNITS) {
    e.push_back({"&bode::rk_step_rt_kernel<" + F(0) + ">", &p->rk});
    e.push_back({"&bode::initial_step_kernel<" + F(0) + ">", &p->initial});
  }
  return e;
}

// compile (or fetch from the cache) the cubin and the lowered kernel names
int build(bode_program* p, const std::string& user, std::string& cubin,
          std::vector<std::string>& lowered) {
  const Nvrtc& N = nvrtc();
  if (!N.ok) return set_error(BODE_EUNSUPPORTED, "bode_program_create: " + N.why);
  int vmaj = 0, vmin = 0;
  N.version(&vmaj, &vmin);
  const std::vector<Entry> ents = entries(p);
  std::string src = "#include \"bode_program.cuh\"\n";
  src += user;
  src += "\n";
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-default-device",
                        "-lineinfo", "-DBODE_RTC_PROGRAM=1"};
  const int nopt = (int)(sizeof(opts) / sizeof(opts[0]));
  std::string key = src + "\n" + bode_rtc::kDigest + "\n" + std::to_string(vmaj) + "." +
                    std::to_string(vmin);
  for (const Entry& e : ents) key += "\n" + e.expr;
  for (const char* o : opts) key += std::string("\n") + o;
  char hex[17];
  snprintf(hex, sizeof hex, "%016llx", (unsigned long long)fnv1a(key));
  const std::string dir = cache_dir(), base = dir + "/" + hex;
  std::string names;
  if (read_file(base + ".cubin", cubin) && read_file(base + ".names", names)) {
    lowered.clear();
    size_t s = 0, q;
    while ((q = names.find('\n', s)) != std::string::npos) {
      lowered.push_back(names.substr(s, q - s));
      s = q + 1;
    }
    if (lowered.size() == ents.size()) return BODE_OK;
  }
  void* prog = nullptr;
  if (N.create(&prog, src.c_str(), "bode_program.cu", bode_rtc::kNumHeaders, bode_rtc::kSources,
               bode_rtc::kNames) != 0)
    return set_error(BODE_ECUDA, "nvrtcCreateProgram failed");
  for (const Entry& e : ents) N.add_name(prog, e.expr.c_str());
  const int rc = N.compile(prog, nopt, opts);
  size_t ls = 0;
  N.log_size(prog, &ls);
  std::string log(ls, '\0');
  if (ls) N.log(prog, &log[0]);
  if (rc != 0) {
    N.destroy(&prog);
    return set_error(BODE_EINVAL, "bode_program_create: the generated kernels do not compile:\n" + log);
  }
  size_t cs = 0;
  N.cubin_size(prog, &cs);
  cubin.assign(cs, '\0');
  N.cubin(prog, &cubin[0]);
  lowered.clear();
  names.clear();
  for (const Entry& e : ents) {
    const char* ln = nullptr;
    N.lowered(prog, e.expr.c_str(), &ln);
    lowered.push_back(ln ? ln : "");
    names += lowered.back() + "\n";
  }
  N.destroy(&prog);
  mkdirs(dir);
  write_file_atomic(base + ".names", names);
  write_file_atomic(base + ".cubin", cubin);
  return BODE_OK;
}

unsigned grid_for(int64_t n) { return (unsigned)((n + 127) / 128); }

cudaError_t launch(CUfunction f, unsigned grid, unsigned block, unsigned smem, cudaStream_t st,
                   void** args) {
  if (!f) return cudaErrorNotSupported;
  return as_cuda(driver().launch(f, grid, 1, 1, block, 1, 1, smem, (CUstream)st, args, nullptr));
}

}  // namespace

const bode_program_desc& program_desc(const bode_program* p) { return p->desc; }

cudaError_t program_init(const bode_program* p, int mode, const SolveParams& P, cudaStream_t st) {
  const int m = mode == BODE_MODE_FAST ? 1 : 0;
  const int64_t ib = (P.n + 127) / 128;
  void* args[] = {(void*)&P};
  return launch(p->init[m], (unsigned)(ib < 148 * 64 ? ib : 148 * 64), 128, 0, st, args);
}

// launch_persistent (bode_solver.cuh) through the driver API
cudaError_t program_solve(const bode_program* p, int mode, const SolveParams& P, int threads,
                          int blocks, cudaStream_t st) {
  const int m = mode == BODE_MODE_FAST ? 1 : 0;
  const bool pi = m == 1 && P.ctrl.plain_pi;
  CUfunction kern = pi ? p->solve_pi : p->solve[m];
  if (!kern || !p->init[m]) return cudaErrorNotSupported;
  const Driver& D = driver();
  const size_t smem = (size_t)P.smem_words * 4;
  if (smem > 48 * 1024) {
    const cudaError_t e = as_cuda(D.set_attr(kern, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem));
    if (e != cudaSuccess) return e;
  }
  if (threads <= 0) threads = 128;
  if (threads > 128 || threads % 32) return cudaErrorInvalidConfiguration;
  if (blocks <= 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    D.occupancy(&per_sm, kern, threads, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t need = (P.n + threads - 1) / threads;
    blocks = (int)((int64_t)sms * per_sm < need ? (int64_t)sms * per_sm : need);
    if (blocks < 1) blocks = 1;
  }
  cudaError_t e = program_init(p, mode, P, st);
  if (e != cudaSuccess) return e;
  if (P.ev_start) cudaEventRecord((cudaEvent_t)P.ev_start, st);
  void* args[] = {(void*)&P};
  e = launch(kern, (unsigned)blocks, (unsigned)threads, (unsigned)smem, st, args);
  if (P.ev_stop) cudaEventRecord((cudaEvent_t)P.ev_stop, st);
  return e;
}

cudaError_t program_joint(const bode_program* p, int mode, const SolveParams& P, const JointWs& W,
                          cudaStream_t st) {
  void* args[] = {(void*)&P, (void*)&W};
  return launch(p->joint[mode == BODE_MODE_FAST ? 1 : 0], 1, kJT, 0, st, args);
}

cudaError_t program_step(const bode_program* p, int mode, const SolveParams& P,
                         const StepState& S, cudaStream_t st) {
  void* args[] = {(void*)&P, (void*)&S};
  return launch(p->step[mode == BODE_MODE_FAST ? 1 : 0], grid_for(P.n), 128, 0, st, args);
}

cudaError_t program_rk_step(const bode_program* p, const bode_tableau* tab, const DynParams& dp,
                            int64_t n, const double* t, const double* dt, const double* y,
                            const double* f0, double* yn, double* err, double* k,
                            cudaStream_t st) {
  void* args[] = {(void*)&dp, &tab, &n, &t, &dt, &y, &f0, &yn, &err, &k};
  return launch(p->rk, grid_for(n), 128, 0, st, args);
}

cudaError_t program_initial_step(const bode_program* p, const DynParams& dp, int64_t n,
                                 const double* t0, const double* y0, int order, const double* av,
                                 const double* rv, double a, double r, const double* dir,
                                 double* dt, double* f0, cudaStream_t st) {
  void* args[] = {(void*)&dp, &n, &t0, &y0, &order, &av, &rv, &a, &r, &dir, &dt, &f0};
  return launch(p->initial, grid_for(n), 128, 0, st, args);
}

}  // namespace bode

namespace {
int check_desc(const char* source, const bode_program_desc* desc) {
  using namespace bode;
  if (!source || !desc) return set_error(BODE_EINVAL, "bode_program_create: null argument");
  if (desc->method < BODE_METHOD_DOPRI5 || desc->method > BODE_METHOD_CUSTOM)
    return set_error(BODE_EINVAL, "bode_program_create: unknown method");
  if (desc->d < 1 || desc->d > 64)
    return set_error(BODE_EUNSUPPORTED, "bode_program_create: state width must be in [1, 64]");
  if (desc->n_params < 0) return set_error(BODE_EINVAL, "bode_program_create: n_params < 0");
  if (desc->method == BODE_METHOD_CUSTOM &&
      (desc->stages < 1 || desc->stages > 16 || desc->error_order < 0 || desc->order < 1))
    return set_error(BODE_EINVAL, "bode_program_create: invalid tableau metadata");
  if (!(desc->kernels & (BODE_PROGRAM_SOLVE | BODE_PROGRAM_STEP | BODE_PROGRAM_UNITS | BODE_PROGRAM_JOINT)))
    return set_error(BODE_EINVAL, "bode_program_create: empty kernel mask");
  return BODE_OK;
}
}  // namespace

extern "C" int bode_program_check(const char* source, const bode_program_desc* desc) {
  using namespace bode;
  int rc = check_desc(source, desc);
  if (rc != BODE_OK) return rc;
  bode_program p;
  p.desc = *desc;
  std::string cubin;
  std::vector<std::string> lowered;
  return build(&p, source, cubin, lowered);
}

extern "C" int bode_program_create(const char* source, const bode_program_desc* desc,
                                   bode_program** out) {
  using namespace bode;
  if (!out) return set_error(BODE_EINVAL, "bode_program_create: null argument");
  *out = nullptr;
  int rc0 = check_desc(source, desc);
  if (rc0 != BODE_OK) return rc0;
  const Driver& D = driver();
  if (!D.ok) return set_error(BODE_ECUDA, "bode_program_create: CUDA driver entry points unavailable");
  bode_program* p = new bode_program;
  p->desc = *desc;
  std::string cubin;
  std::vector<std::string> lowered;
  int rc = build(p, source, cubin, lowered);
  if (rc != BODE_OK) {
    delete p;
    return rc;
  }
  cudaFree(nullptr);  // make sure the device's primary context is current
  CUresult r = D.load(&p->mod, cubin.data());
  if (r != CUDA_SUCCESS) {
    delete p;
    return set_error(BODE_ECUDA, "bode_program_create: cuModuleLoadData failed (" +
                                     std::to_string((int)r) + ")");
  }
  const std::vector<Entry> ents = entries(p);
  for (size_t k = 0; k < ents.size(); k++) {
    r = D.get_function(ents[k].slot, p->mod, lowered[k].c_str());
    if (r != CUDA_SUCCESS) {
      D.unload(p->mod);
      delete p;
      return set_error(BODE_ECUDA, "bode_program_create: kernel " + ents[k].expr + " missing");
    }
  }
  *out = p;
  return BODE_OK;
}

extern "C" void bode_program_destroy(bode_program* prog) {
  if (!prog) return;
  if (prog->mod) bode::driver().unload(prog->mod);
  delete prog;
}
