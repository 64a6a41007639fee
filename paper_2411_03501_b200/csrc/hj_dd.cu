// hj_dd.cu -- multi-GPU slab decomposition of the fused stage,
// NCCL over NVLink behind the C ABI (include/hjb200.h, hj_dd_*).
//
// Axis 0 of the grid is split into contiguous slabs, one per rank (one
// process per GPU).  A rank's field buffer carries hj_grid.halo exchanged
// planes in front of and behind its owned planes.  Per RK stage:
//   1. the caller's stream records "input ready"; the communicator's stream
//      waits on it and runs ONE grouped ncclSend/ncclRecv of the boundary
//      planes with each neighbour (the reference's ghost extension along
//      axis 0, grid.py:203-225, becomes a copy of the neighbour's planes);
//   2. meanwhile the CORE part of the stage (the brick rows whose stencils
//      read no exchanged plane, hj_stage_part) runs on the caller's stream;
//   3. the caller's stream waits on the exchange (no host synchronisation)
//      and the RIM part runs.
// CORE + RIM is the same set of node updates as one launch and the halos
// are exact copies, so the decomposed result is bit-identical to one GPU.
// Per interval the non-finite flags / first failing stage / costate ranges
// are all-reduced (hj_dd_reduce_stats), so every rank raises the error the
// single-GPU run raises; snapshots are gathered to a root (hj_dd_gather).
//
// libnccl is resolved at run time (dlopen of libnccl.so.2 -- inside a torch
// process that is the copy torch already loaded), so the library has no
// link-time NCCL dependency and loads on hosts without it.
#include <dlfcn.h>
#include <nccl.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include "hj_kernels.cuh"

namespace hj {
int set_error(int code, const char* msg);
void count_launches(uint64_t n);
bool axes_slab_applies(const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha, int stage,
                       const double* y_in, const double* y0, double* y_out);
int stage_axes_part(const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha, double dt, int stage,
                    const double* y_in, const double* y0, double* y_out, const double* mask_prev, int mask,
                    hj_stats* stats, int32_t tag, int which, void* stream);
}  // namespace hj

using namespace hj;

namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  int version = 0;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi load_nccl() {
  NcclApi a;
  const char* env = std::getenv("HJ_NCCL_LIB");
  void* h = dlopen(env && *env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    a.why = std::string("cannot load NCCL: ") + dlerror();
    return a;
  }
#define HJ_SYM(field, name)                                            \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name));       \
  if (!a.field) {                                                      \
    a.why = std::string("NCCL library lacks ") + name;                 \
    return a;                                                          \
  }
  HJ_SYM(GetVersion, "ncclGetVersion");
  HJ_SYM(GetUniqueId, "ncclGetUniqueId");
  HJ_SYM(CommInitRank, "ncclCommInitRank");
  HJ_SYM(CommDestroy, "ncclCommDestroy");
  HJ_SYM(GroupStart, "ncclGroupStart");
  HJ_SYM(GroupEnd, "ncclGroupEnd");
  HJ_SYM(Send, "ncclSend");
  HJ_SYM(Recv, "ncclRecv");
  HJ_SYM(AllReduce, "ncclAllReduce");
  HJ_SYM(GetErrorString, "ncclGetErrorString");
#undef HJ_SYM
  a.GetVersion(&a.version);
  a.ok = true;
  return a;
}

const NcclApi& nccl() {
  static std::once_flag once;
  static NcclApi api;
  std::call_once(once, [] { api = load_nccl(); });
  return api;
}

int nccl_fail(ncclResult_t r, const char* what) {
  char buf[384];
  std::snprintf(buf, sizeof buf, "%s: %s", what, nccl().GetErrorString ? nccl().GetErrorString(r) : "NCCL error");
  return set_error(HJ_ENCCL, buf);
}

int cuda_fail(cudaError_t e, const char* what) {
  char buf[384];
  std::snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
  return set_error(HJ_ECUDA, buf);
}

int inval(const char* msg) { return set_error(HJ_EINVAL, msg); }

#define HJ_NCCL(call, what)                      \
  do {                                           \
    ncclResult_t r_ = (call);                    \
    if (r_ != ncclSuccess) return nccl_fail(r_, what); \
  } while (0)
#define HJ_CUDA(call, what)                      \
  do {                                           \
    cudaError_t e_ = (call);                     \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

// hj_stats.nonfinite is a bit set (OR-reduced); NCCL has no OR, so the bits
// travel as one int32 each and are max-reduced.
constexpr int NBITS = 8;

__global__ void k_stats_unpack_bits(const hj_stats* st, int* bits) {
  const int b = threadIdx.x;
  if (b < NBITS) bits[b] = (st->nonfinite >> b) & 1u;
}

__global__ void k_stats_pack_bits(hj_stats* st, const int* bits) {
  if (threadIdx.x == 0) {
    unsigned f = 0u;
    for (int b = 0; b < NBITS; ++b) f |= bits[b] ? (1u << b) : 0u;
    st->nonfinite = f;
  }
}

}  // namespace

struct hj_dd {
  ncclComm_t comm = nullptr;
  int nranks = 0, rank = 0, device = 0;
  int lo_rank = -1, hi_rank = -1;      // neighbours along axis 0 (-1: global edge)
  cudaStream_t comm_stream = nullptr;  // halo exchange runs here, overlapped with CORE
  cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
  int* d_bits = nullptr;
  uint64_t exchanges = 0, halo_bytes = 0;
};

extern "C" {

int hj_dd_nccl_version(void) {
  const NcclApi& a = nccl();
  if (!a.ok) return set_error(HJ_ENCCL, a.why.c_str());
  return a.version;
}

int hj_dd_unique_id(void* uid) {
  if (!uid) return inval("uid is NULL");
  const NcclApi& a = nccl();
  if (!a.ok) return set_error(HJ_ENCCL, a.why.c_str());
  ncclUniqueId id;
  HJ_NCCL(a.GetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == HJ_DD_UID_BYTES, "unique id size");
  std::memcpy(uid, &id, sizeof id);
  return HJ_OK;
}

int hj_dd_init(const void* uid, int nranks, int rank, int lo_rank, int hi_rank, hj_dd** out) {
  if (!uid || !out) return inval("NULL argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return inval("rank out of range");
  if (lo_rank < -1 || lo_rank >= nranks || hi_rank < -1 || hi_rank >= nranks) return inval("neighbour rank out of range");
  const NcclApi& a = nccl();
  if (!a.ok) return set_error(HJ_ENCCL, a.why.c_str());
  hj_dd* dd = new hj_dd;
  dd->nranks = nranks;
  dd->rank = rank;
  dd->lo_rank = lo_rank;
  dd->hi_rank = hi_rank;
  cudaGetDevice(&dd->device);
  int lo_prio = 0, hi_prio = 0;
  cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
  cudaError_t e = cudaStreamCreateWithPriority(&dd->comm_stream, cudaStreamNonBlocking, hi_prio);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&dd->ev_ready, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&dd->ev_halo, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaMalloc((void**)&dd->d_bits, NBITS * sizeof(int));
  if (e != cudaSuccess) {
    hj_dd_free(dd);
    return cuda_fail(e, "hj_dd_init");
  }
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof id);
  ncclResult_t r = a.CommInitRank(&dd->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    dd->comm = nullptr;
    hj_dd_free(dd);
    return nccl_fail(r, "ncclCommInitRank");
  }
  *out = dd;
  return HJ_OK;
}

int hj_dd_free(hj_dd* dd) {
  if (!dd) return HJ_OK;
  if (dd->comm_stream) cudaStreamSynchronize(dd->comm_stream);
  if (dd->comm) nccl().CommDestroy(dd->comm);
  if (dd->ev_ready) cudaEventDestroy(dd->ev_ready);
  if (dd->ev_halo) cudaEventDestroy(dd->ev_halo);
  if (dd->comm_stream) cudaStreamDestroy(dd->comm_stream);
  if (dd->d_bits) cudaFree(dd->d_bits);
  delete dd;
  return HJ_OK;
}

// Post the halo exchange of `buf` (pointer at the first owned plane) on the
// communicator's stream, ordered after the work queued on `stream`.
// Message order: sends [to lower, to upper], receives [from upper, from
// lower] -- the k-th message from A to B then pairs with B's k-th receive
// from A even when both neighbours are the same rank (a two-slab periodic
// ring) or this rank itself (a one-slab periodic ring).
static int post_exchange(hj_dd* dd, const hj_grid* g, const double* buf, cudaStream_t stream) {
  const NcclApi& a = nccl();
  long long plane = 1;
  for (int ax = 1; ax < g->dim; ++ax) plane *= g->n[ax];
  const size_t cnt = (size_t)(g->halo * plane);
  const long long n0 = g->n[0];
  double* b = const_cast<double*>(buf);
  HJ_CUDA(cudaEventRecord(dd->ev_ready, stream), "hj_dd_stage: cudaEventRecord");
  HJ_CUDA(cudaStreamWaitEvent(dd->comm_stream, dd->ev_ready, 0), "hj_dd_stage: cudaStreamWaitEvent");
  HJ_NCCL(a.GroupStart(), "ncclGroupStart");
  if (g->halo_lo) HJ_NCCL(a.Send(b, cnt, ncclFloat64, dd->lo_rank, dd->comm, dd->comm_stream), "ncclSend");
  if (g->halo_hi)
    HJ_NCCL(a.Send(b + (n0 - g->halo) * plane, cnt, ncclFloat64, dd->hi_rank, dd->comm, dd->comm_stream), "ncclSend");
  if (g->halo_hi) HJ_NCCL(a.Recv(b + n0 * plane, cnt, ncclFloat64, dd->hi_rank, dd->comm, dd->comm_stream), "ncclRecv");
  if (g->halo_lo) HJ_NCCL(a.Recv(b - g->halo * plane, cnt, ncclFloat64, dd->lo_rank, dd->comm, dd->comm_stream), "ncclRecv");
  HJ_NCCL(a.GroupEnd(), "ncclGroupEnd");
  HJ_CUDA(cudaEventRecord(dd->ev_halo, dd->comm_stream), "hj_dd_stage: cudaEventRecord");
  dd->exchanges += 1;
  dd->halo_bytes += (size_t)((g->halo_lo ? 1 : 0) + (g->halo_hi ? 1 : 0)) * cnt * sizeof(double);
  return HJ_OK;
}

int hj_dd_stage(hj_dd* dd, const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha, double dt,
                int stage, const double* y_in, const double* y0, double* y_out, const double* mask_prev, int mask,
                hj_stats* stats, int32_t tag, int overlap, void* stream) {
  if (!dd || !g) return inval("NULL argument");
  if (g->batch != 1) return inval("slab stages take one problem (batch 1)");
  if ((g->halo_lo && dd->lo_rank < 0) || (g->halo_hi && dd->hi_rank < 0))
    return inval("grid expects a halo from a neighbour the communicator does not have");
  if ((g->halo_lo || g->halo_hi) && g->halo < HJ_HALO_MIN) return inval("slab halo thinner than HJ_HALO_MIN planes");
  if ((g->halo_lo || g->halo_hi) && g->n[0] < g->halo) return inval("slab holds fewer planes than its halo");
  if (!y_in) return inval("NULL field pointer");
  cudaStream_t s = (cudaStream_t)stream;
  if (!g->halo_lo && !g->halo_hi)
    return hj_stage(g, scheme, ham, alpha, dt, stage, y_in, y0, y_out, mask_prev, mask, stats, tag, stream);
  // per-axis walk pipeline (large WENO5 slabs): only the axis-0 walk reads
  // exchanged planes, so the contiguous-axis kernel overlaps the exchange and
  // the column kernels follow it -- no CORE/RIM split
  if (overlap && axes_slab_applies(g, scheme, ham, alpha, stage, y_in, y0, y_out)) {
    int rc = post_exchange(dd, g, y_in, s);
    if (rc) return rc;
    rc = stage_axes_part(g, scheme, ham, alpha, dt, stage, y_in, y0, y_out, mask_prev, mask, stats, tag, 1, stream);
    if (rc) return rc;
    HJ_CUDA(cudaStreamWaitEvent(s, dd->ev_halo, 0), "hj_dd_stage: cudaStreamWaitEvent");
    return stage_axes_part(g, scheme, ham, alpha, dt, stage, y_in, y0, y_out, mask_prev, mask, stats, tag, 2, stream);
  }
  int rc = post_exchange(dd, g, y_in, s);
  if (rc) return rc;
  if (overlap) {
    rc = hj_stage_part(g, scheme, ham, alpha, dt, stage, y_in, y0, y_out, mask_prev, mask, stats, tag,
                       HJ_PART_CORE, stream);
    if (rc) return rc;
  }
  HJ_CUDA(cudaStreamWaitEvent(s, dd->ev_halo, 0), "hj_dd_stage: cudaStreamWaitEvent");
  return hj_stage_part(g, scheme, ham, alpha, dt, stage, y_in, y0, y_out, mask_prev, mask, stats, tag,
                       overlap ? HJ_PART_RIM : HJ_PART_ALL, stream);
}

int hj_dd_exchange(hj_dd* dd, const hj_grid* g, double* buf, void* stream) {
  if (!dd || !g || !buf) return inval("NULL argument");
  if ((g->halo_lo && dd->lo_rank < 0) || (g->halo_hi && dd->hi_rank < 0))
    return inval("grid expects a halo from a neighbour the communicator does not have");
  if (!g->halo_lo && !g->halo_hi) return HJ_OK;
  int rc = post_exchange(dd, g, buf, (cudaStream_t)stream);
  if (rc) return rc;
  HJ_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, dd->ev_halo, 0), "hj_dd_exchange");
  return HJ_OK;
}

int hj_dd_reduce_stats(hj_dd* dd, hj_stats* stats, void* stream) {
  if (!dd || !stats) return inval("NULL argument");
  const NcclApi& a = nccl();
  cudaStream_t s = (cudaStream_t)stream;
  k_stats_unpack_bits<<<1, 32, 0, s>>>(stats, dd->d_bits);
  HJ_CUDA(cudaGetLastError(), "hj_dd_reduce_stats");
  HJ_NCCL(a.GroupStart(), "ncclGroupStart");
  HJ_NCCL(a.AllReduce(stats->lo_key, stats->lo_key, HJ_MAX_DIM, ncclInt64, ncclMin, dd->comm, s), "ncclAllReduce");
  HJ_NCCL(a.AllReduce(stats->hi_key, stats->hi_key, HJ_MAX_DIM, ncclInt64, ncclMax, dd->comm, s), "ncclAllReduce");
  HJ_NCCL(a.AllReduce(dd->d_bits, dd->d_bits, NBITS, ncclInt32, ncclMax, dd->comm, s), "ncclAllReduce");
  HJ_NCCL(a.AllReduce(&stats->first_bad_tag, &stats->first_bad_tag, 1, ncclInt32, ncclMin, dd->comm, s),
          "ncclAllReduce");
  HJ_NCCL(a.GroupEnd(), "ncclGroupEnd");
  k_stats_pack_bits<<<1, 32, 0, s>>>(stats, dd->d_bits);
  HJ_CUDA(cudaGetLastError(), "hj_dd_reduce_stats");
  count_launches(2);
  return HJ_OK;
}

int hj_dd_gather(hj_dd* dd, const double* owned, int64_t count, double* full, const int64_t* counts, int root,
                 void* stream) {
  if (!dd || !owned) return inval("NULL argument");
  if (root < 0 || root >= dd->nranks) return inval("root out of range");
  const NcclApi& a = nccl();
  cudaStream_t s = (cudaStream_t)stream;
  if (dd->rank != root) {
    HJ_NCCL(a.Send(owned, (size_t)count, ncclFloat64, root, dd->comm, s), "ncclSend");
    return HJ_OK;
  }
  if (!full || !counts) return inval("root needs the full buffer and the per-rank counts");
  if (counts[root] != count) return inval("root's count disagrees with counts[root]");
  int64_t off = 0;
  HJ_NCCL(a.GroupStart(), "ncclGroupStart");
  for (int r = 0; r < dd->nranks; ++r) {
    if (r == root) {
      if (count)
        HJ_CUDA(cudaMemcpyAsync(full + off, owned, (size_t)count * sizeof(double), cudaMemcpyDeviceToDevice, s),
                "hj_dd_gather: cudaMemcpyAsync");
    } else {
      HJ_NCCL(a.Recv(full + off, (size_t)counts[r], ncclFloat64, r, dd->comm, s), "ncclRecv");
    }
    off += counts[r];
  }
  HJ_NCCL(a.GroupEnd(), "ncclGroupEnd");
  return HJ_OK;
}

int hj_dd_stats(const hj_dd* dd, uint64_t* exchanges, uint64_t* halo_bytes) {
  if (!dd) return inval("NULL argument");
  if (exchanges) *exchanges = dd->exchanges;
  if (halo_bytes) *halo_bytes = dd->halo_bytes;
  return HJ_OK;
}

}  // extern "C"
