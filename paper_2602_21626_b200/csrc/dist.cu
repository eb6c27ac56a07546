// NCCL for the multi-GPU form of the pass: token shards per rank, an in-place SUM
// all-reduce of the u64 counts, candidate slices per rank and a MIN merge of the objectives.
//
// The library does not link NCCL.  Its entry points are resolved at first use from the libnccl.so.2
// already mapped into the process (the one that created a caller's communicator, e.g. torch's
// ProcessGroupNCCL, whose ncclComm_t is then used as is), else loaded from the system.  Types come
// from the NCCL header only.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstdint>
#include <string>

#include "internal.cuh"

namespace gimbal_gpu {

namespace {

struct NcclApi {
  void* so = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*comm_count)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*comm_user_rank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string why;
};

const NcclApi& api() {
  static const NcclApi a = [] {
    NcclApi r;
    r.so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's NCCL, if any
    if (!r.so) r.so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!r.so) {
      const char* e = dlerror();
      r.why = std::string("libnccl.so.2 not loadable: ") + (e ? e : "?");
      return r;
    }
    auto sym = [&](const char* n) { return dlsym(r.so, n); };
    r.get_unique_id = reinterpret_cast<decltype(r.get_unique_id)>(sym("ncclGetUniqueId"));
    r.comm_init_rank = reinterpret_cast<decltype(r.comm_init_rank)>(sym("ncclCommInitRank"));
    r.comm_destroy = reinterpret_cast<decltype(r.comm_destroy)>(sym("ncclCommDestroy"));
    r.comm_count = reinterpret_cast<decltype(r.comm_count)>(sym("ncclCommCount"));
    r.comm_user_rank = reinterpret_cast<decltype(r.comm_user_rank)>(sym("ncclCommUserRank"));
    r.all_reduce = reinterpret_cast<decltype(r.all_reduce)>(sym("ncclAllReduce"));
    r.error_string = reinterpret_cast<decltype(r.error_string)>(sym("ncclGetErrorString"));
    if (!r.get_unique_id || !r.comm_init_rank || !r.comm_destroy || !r.comm_count || !r.all_reduce)
      r.why = "libnccl.so.2 lacks an expected symbol";
    return r;
  }();
  return a;
}

int nccl_fail(const char* what, ncclResult_t r) {
  const NcclApi& a = api();
  set_error(std::string(what) + ": " + (a.error_string ? a.error_string(r) : "NCCL error"));
  return GIMBAL_NCCL_ERROR;
}

int need_api() {
  if (!api().why.empty()) {
    set_error(api().why);
    return GIMBAL_NCCL_ERROR;
  }
  return GIMBAL_OK;
}

// objectives of this rank's slice -> [n_total] vector (+inf elsewhere) for the MIN all-reduce
__global__ void scatter_slice_kernel(const double* __restrict__ local, int64_t n_local, int64_t offset,
                                     double* __restrict__ global, int64_t n_total) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = i - offset;
    global[i] = (j >= 0 && j < n_local) ? local[j] : __longlong_as_double(0x7ff0000000000000ll);
  }
}

// lowest index among the minimal objectives (the placement argmin tie rule)
__global__ void argmin_kernel(const double* __restrict__ v, int64_t n, long long* __restrict__ out) {
  __shared__ double bv[1024];
  __shared__ long long bi[1024];
  double best = 0.0;
  long long besti = -1;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
    if (besti < 0 || v[i] < best) {
      best = v[i];
      besti = i;
    }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = besti;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double v2 = bv[threadIdx.x + s];
      const long long i2 = bi[threadIdx.x + s], i1 = bi[threadIdx.x];
      if (i2 >= 0 && (i1 < 0 || v2 < bv[threadIdx.x] || (v2 == bv[threadIdx.x] && i2 < i1))) {
        bv[threadIdx.x] = v2;
        bi[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = bi[0];
}

}  // namespace

int nccl_allreduce_u64_sum(unsigned long long* buf, size_t n, void* comm, cudaStream_t s) {
  GIMBAL_TRY(need_api());
  // ncclUint64 SUM is plain u64 addition: bit-identical in any order
  const ncclResult_t r = api().all_reduce(buf, buf, n, ncclUint64, ncclSum, static_cast<ncclComm_t>(comm), s);
  return r == ncclSuccess ? GIMBAL_OK : nccl_fail("ncclAllReduce(counts)", r);
}

int nccl_merge_argmin(const double* local, int64_t n_local, int64_t offset, double* global, int64_t n_total,
                      long long* argmin, void* comm, cudaStream_t s) {
  GIMBAL_TRY(need_api());
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(1184, (n_total + 255) / 256));
  scatter_slice_kernel<<<grid, 256, 0, s>>>(local, n_local, offset, global, n_total);
  GIMBAL_CUDA_TRY(cudaGetLastError());
  const ncclResult_t r = api().all_reduce(global, global, (size_t)n_total, ncclFloat64, ncclMin,
                                          static_cast<ncclComm_t>(comm), s);
  if (r != ncclSuccess) return nccl_fail("ncclAllReduce(objectives)", r);
  argmin_kernel<<<1, 1024, 0, s>>>(global, n_total, argmin);
  GIMBAL_CUDA_TRY(cudaGetLastError());
  return GIMBAL_OK;
}

}  // namespace gimbal_gpu

using namespace gimbal_gpu;

extern "C" {

int gimbal_dist_unique_id(void* unique_id) {
  if (!unique_id) return invalid("gimbal_dist_unique_id: null output");
  GIMBAL_TRY(need_api());
  ncclUniqueId id;
  const ncclResult_t r = api().get_unique_id(&id);
  if (r != ncclSuccess) return nccl_fail("ncclGetUniqueId", r);
  static_assert(sizeof(ncclUniqueId) == GIMBAL_DIST_UNIQUE_ID_BYTES, "ncclUniqueId size");
  memcpy(unique_id, &id, sizeof(id));
  return GIMBAL_OK;
}

int gimbal_dist_comm_init(int32_t n_ranks, int32_t rank, const void* unique_id, int device, gimbal_comm_t* out) {
  if (!unique_id || !out) return invalid("gimbal_dist_comm_init: null argument");
  if (n_ranks < 1 || rank < 0 || rank >= n_ranks) return invalid("gimbal_dist_comm_init: rank out of range");
  GIMBAL_TRY(need_api());
  DeviceGuard g(device);
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  ncclComm_t c = nullptr;
  const ncclResult_t r = api().comm_init_rank(&c, n_ranks, id, rank);
  if (r != ncclSuccess) return nccl_fail("ncclCommInitRank", r);
  *out = c;
  return GIMBAL_OK;
}

int gimbal_dist_comm_destroy(gimbal_comm_t comm) {
  if (!comm) return GIMBAL_OK;
  GIMBAL_TRY(need_api());
  const ncclResult_t r = api().comm_destroy(static_cast<ncclComm_t>(comm));
  return r == ncclSuccess ? GIMBAL_OK : nccl_fail("ncclCommDestroy", r);
}

int gimbal_dist_comm_size(gimbal_comm_t comm, int32_t* n_ranks, int32_t* rank) {
  if (!comm) return invalid("gimbal_dist_comm_size: null communicator");
  GIMBAL_TRY(need_api());
  int n = 0, r = 0;
  ncclResult_t st = api().comm_count(static_cast<ncclComm_t>(comm), &n);
  if (st != ncclSuccess) return nccl_fail("ncclCommCount", st);
  if (api().comm_user_rank) {
    st = api().comm_user_rank(static_cast<ncclComm_t>(comm), &r);
    if (st != ncclSuccess) return nccl_fail("ncclCommUserRank", st);
  }
  if (n_ranks) *n_ranks = n;
  if (rank) *rank = r;
  return GIMBAL_OK;
}

}  // extern "C"
