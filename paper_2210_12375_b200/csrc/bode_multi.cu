// bode_multi.cu -- bode_solve_multi (include/bode.h): one batch sharded
// across the GPUs of one process (SURVEY.md 8(b) "bode_solve_multi", 8(e)).
//
// Every shard is an independent bode_solve on its own device and stream
// (instances are independent: a shard is bitwise equal to its rows of the
// full batch, tests/test_solver.py:140-168).  The one quantity that couples
// the shards is the reference's batch-global n_f_evals (solver.py:184,224,
// 239): 1 + (S-1) max_i n_steps_i + #{iterations j >= 1 in which some
// running row had rejected at j-1} for FSAL tableaus, 1 + S max_i n_steps_i
// otherwise.  Each shard reports its largest n_steps and its per-iteration
// refresh bytes (max_iterations_out / refresh_map_out); the combine is a MAX
// of both across shards -- an NCCL all-reduce over NVLink when the caller
// passes communicators, else one kernel on the first shard's device reading
// every shard's buffers through peer access -- and every shard's n_f_evals,
// max_iterations_out and refresh_map_out then hold the batch-global values.
// NCCL is resolved at run time (dlopen), so libbode.so has no link-time
// dependency on it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdint>
#include <string>

#include "../../include/bode.h"

namespace bode {
int set_error(int code, const std::string& msg);
}

namespace {

constexpr int kMaxShards = 16;

struct Shards {
  int64_t* mx[kMaxShards];
  uint8_t* map[kMaxShards];
  int64_t* nfe[kMaxShards];
  int ndev;
  int64_t len;
  int stages, fsal;
};

// one CTA: global max of n_steps, OR of the refresh bytes, the count, and
// the batch-global values written back to every shard
__global__ void combine_kernel(Shards S) {
  __shared__ int64_t s_mx;
  __shared__ unsigned long long s_cnt;
  if (threadIdx.x == 0) {
    int64_t m = 0;
    for (int k = 0; k < S.ndev; k++) m = *S.mx[k] > m ? *S.mx[k] : m;
    s_mx = m;
    s_cnt = 0;
  }
  __syncthreads();
  const int64_t mx = s_mx;
  unsigned long long cnt = 0;
  for (int64_t j = threadIdx.x; j < S.len; j += blockDim.x) {
    uint8_t v = 0;
    for (int k = 0; k < S.ndev; k++) v |= S.map[k][j];
    if (S.ndev > 1)
      for (int k = 0; k < S.ndev; k++) S.map[k][j] = v;
    if (v && j >= 1 && j < mx) cnt++;
  }
  atomicAdd(&s_cnt, cnt);
  __syncthreads();
  if (threadIdx.x == 0) {
    const int64_t total = S.fsal ? 1 + (int64_t)(S.stages - 1) * mx + (int64_t)s_cnt
                                 : 1 + (int64_t)S.stages * mx;
    for (int k = 0; k < S.ndev; k++) {
      *S.mx[k] = mx;
      *S.nfe[k] = total;
    }
  }
}

struct Nccl {
  ncclResult_t (*group_start)();
  ncclResult_t (*group_end)();
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t);
  const char* (*error_string)(ncclResult_t);
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl r;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return r;
    r.group_start = (decltype(r.group_start))dlsym(h, "ncclGroupStart");
    r.group_end = (decltype(r.group_end))dlsym(h, "ncclGroupEnd");
    r.all_reduce = (decltype(r.all_reduce))dlsym(h, "ncclAllReduce");
    r.error_string = (decltype(r.error_string))dlsym(h, "ncclGetErrorString");
    r.ok = r.group_start && r.group_end && r.all_reduce && r.error_string;
    return r;
  }();
  return n;
}

int device_of(const void* p, int* dev) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess || at.type != cudaMemoryTypeDevice) {
    cudaGetLastError();
    return BODE_EINVAL;
  }
  *dev = at.device;
  return BODE_OK;
}

int stages_fsal(const bode_solve_args& a, int* stages, int* fsal) {
  if (a.method == BODE_METHOD_CUSTOM) return BODE_EUNSUPPORTED;
  *stages = a.method == BODE_METHOD_HEUN ? 2 : 7;
  *fsal = a.method == BODE_METHOD_HEUN ? 0 : 1;
  return BODE_OK;
}

}  // namespace

extern "C" int bode_solve_multi(const bode_solve_args* per_dev, int32_t ndev, void* const* comms) {
  using bode::set_error;
  if (!per_dev || ndev < 1) return set_error(BODE_EINVAL, "bode_solve_multi: need at least one shard");
  if (ndev > kMaxShards) return set_error(BODE_EINVAL, "bode_solve_multi: at most 16 shards");
  int stages = 0, fsal = 0;
  if (stages_fsal(per_dev[0], &stages, &fsal) != BODE_OK)
    return set_error(BODE_EUNSUPPORTED, "bode_solve_multi: built-in tableaus only");
  int devs[kMaxShards];
  for (int k = 0; k < ndev; k++) {
    const bode_solve_args& a = per_dev[k];
    if (a.method != per_dev[0].method || a.max_steps != per_dev[0].max_steps)
      return set_error(BODE_EINVAL, "bode_solve_multi: shards must share method and max_steps");
    if (a.joint) return set_error(BODE_EUNSUPPORTED, "bode_solve_multi: independent solves only");
    if (!a.max_iterations_out || !a.refresh_map_out)
      return set_error(BODE_EINVAL,
                       "bode_solve_multi: every shard needs max_iterations_out and refresh_map_out");
    if (!a.y0 || device_of(a.y0, &devs[k]) != BODE_OK)
      return set_error(BODE_EINVAL, "bode_solve_multi: y0 must be a device pointer");
  }
  int prev = 0;
  cudaGetDevice(&prev);
  struct Restore {
    int d;
    ~Restore() { cudaSetDevice(d); }
  } restore{prev};
  // the shard solves, concurrently (stream-ordered, no host sync)
  for (int k = 0; k < ndev; k++) {
    cudaSetDevice(devs[k]);
    const int rc = bode_solve(&per_dev[k]);
    if (rc != BODE_OK) return rc;  // (bode_last_error holds the shard's message)
  }
  const int64_t len = per_dev[0].max_steps + 2;
  if (comms) {  // NCCL: MAX all-reduce over the communicator of these devices
    const Nccl& N = nccl();
    if (!N.ok) return set_error(BODE_EUNSUPPORTED, "bode_solve_multi: libnccl.so.2 not loadable");
    ncclResult_t r = N.group_start();
    for (int k = 0; k < ndev && r == ncclSuccess; k++) {
      cudaSetDevice(devs[k]);
      const bode_solve_args& a = per_dev[k];
      const ncclComm_t c = (ncclComm_t)comms[k];
      cudaStream_t st = (cudaStream_t)a.stream;
      r = N.all_reduce(a.max_iterations_out, a.max_iterations_out, 1, ncclInt64, ncclMax, c, st);
      if (r == ncclSuccess)
        r = N.all_reduce(a.refresh_map_out, a.refresh_map_out, (size_t)len, ncclUint8, ncclMax, c, st);
    }
    const ncclResult_t r2 = N.group_end();
    if (r != ncclSuccess || r2 != ncclSuccess)
      return set_error(BODE_ECUDA, std::string("bode_solve_multi: NCCL: ") +
                                       N.error_string(r != ncclSuccess ? r : r2));
    for (int k = 0; k < ndev; k++) {  // each device counts from its (now global) buffers
      cudaSetDevice(devs[k]);
      const bode_solve_args& a = per_dev[k];
      Shards S{};
      S.mx[0] = a.max_iterations_out, S.map[0] = a.refresh_map_out, S.nfe[0] = a.n_f_evals;
      S.ndev = 1, S.len = len, S.stages = stages, S.fsal = fsal;
      combine_kernel<<<1, 256, 0, (cudaStream_t)a.stream>>>(S);
    }
  } else {  // one kernel on the first shard's device, reading the others by peer access
    for (int k = 1; k < ndev; k++) {
      if (devs[k] == devs[0]) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, devs[0], devs[k]);
      if (!can)
        return set_error(BODE_EUNSUPPORTED,
                         "bode_solve_multi: no peer access between the shards' devices; pass NCCL communicators");
      cudaSetDevice(devs[0]);
      const cudaError_t e = cudaDeviceEnablePeerAccess(devs[k], 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return set_error(BODE_ECUDA, std::string("bode_solve_multi: ") + cudaGetErrorString(e));
      cudaGetLastError();
    }
    Shards S{};
    S.ndev = ndev, S.len = len, S.stages = stages, S.fsal = fsal;
    cudaEvent_t ev[kMaxShards];
    cudaStream_t st0 = (cudaStream_t)per_dev[0].stream;
    for (int k = 0; k < ndev; k++) {
      const bode_solve_args& a = per_dev[k];
      S.mx[k] = a.max_iterations_out, S.map[k] = a.refresh_map_out, S.nfe[k] = a.n_f_evals;
      cudaSetDevice(devs[k]);
      cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming);
      cudaEventRecord(ev[k], (cudaStream_t)a.stream);
      cudaSetDevice(devs[0]);
      cudaStreamWaitEvent(st0, ev[k], 0);
    }
    cudaSetDevice(devs[0]);
    combine_kernel<<<1, 256, 0, st0>>>(S);
    cudaEvent_t done;
    cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
    cudaEventRecord(done, st0);
    for (int k = 0; k < ndev; k++) {  // every shard's stream sees the global values
      cudaSetDevice(devs[k]);
      cudaStreamWaitEvent((cudaStream_t)per_dev[k].stream, done, 0);
      cudaEventDestroy(ev[k]);
    }
    cudaEventDestroy(done);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(BODE_ECUDA, std::string("bode_solve_multi: ") + cudaGetErrorString(e));
  return BODE_OK;
}
