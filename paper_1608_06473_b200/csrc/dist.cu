// Multi-rank support: macro partition, ghost exchange plan, NCCL / host
// transports (PAPER.md:295-302 HHG ghost layers, 853-858).
//
// Every lower-primitive node and every volume node has exactly one owner rank
// (the rank of the lowest-id macro containing it).  The owner computes its row
// and is the source of truth for its value.  A rank additionally stores ghost
// copies of the macros of other ranks that share a vertex with its own.  One
// "sync" moves, for every mirrored slot, the owner's value: ghost-block slots
// read by this rank's rows, and this rank's copies of lower-primitive nodes
// owned elsewhere.  Transport: NCCL point-to-point (ncclGroupStart/Send/Recv,
// device buffers, one process per GPU over NVLink) or, for tests, a host
// callback that moves host buffers (torch.distributed gloo in the binding).
#include <nccl.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <functional>
#include <cstring>
#include <thread>

#include "fem_device.cuh"
#include "hhg_internal.h"

namespace hhg {

typedef int (*HostFn)(void* user, int nranks, const int64_t* send_bytes, const void* send,
                      const int64_t* recv_bytes, void* recv);

static HostFn g_host_fn = nullptr;
static void* g_host_user = nullptr;
static int g_host_only = 0;

#define HHG_NCCL(c, call)                                                                          \
  do {                                                                                             \
    ncclResult_t r__ = (call);                                                                     \
    if (r__ != ncclSuccess) {                                                                      \
      (c)->poisoned = true;                                                                        \
      return set_err(c, HHG_ERR_NCCL, std::string("NCCL: ") + ncclGetErrorString(r__) + " in " #call); \
    }                                                                                              \
  } while (0)

hhg_status dist_init_transport(Ctx* c, const void* nccl_unique_id) {
  if (nccl_unique_id) {
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof(id));
    ncclComm_t comm;
    HHG_NCCL(c, ncclCommInitRank(&comm, c->nranks, id, c->rank));
    c->nccl_comm = comm;
    c->transport = 1;
    return HHG_OK;
  }
  if (!g_host_fn) return set_err(c, HHG_ERR_INVALID, "nranks > 1 needs an NCCL id or hhg_set_host_transport");
  c->host_fn = (void*)g_host_fn;
  c->host_user = g_host_user;
  c->host_only = g_host_only != 0;
  c->transport = 2;
  return HHG_OK;
}

// Wait for the ctx stream; with the NCCL transport, poll the communicator's
// asynchronous error state while waiting and abort it (sticky HHG_ERR_NCCL)
// on an error or after HHG_NCCL_TIMEOUT_S seconds (default 600) without
// progress -- a peer that died must not hang this rank forever.
hhg_status ctx_sync(Ctx* c) {
  if (c->transport != 1 || !c->nccl_comm) {
    HHG_CK(c, cudaStreamSynchronize(c->stream));
    return HHG_OK;
  }
  const char* e = getenv("HHG_NCCL_TIMEOUT_S");
  const double limit = e ? atof(e) : 600.0;
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    cudaError_t q = cudaStreamQuery(c->stream);
    if (q == cudaSuccess) return HHG_OK;
    if (q != cudaErrorNotReady) return check_cuda(c, q, "cudaStreamQuery");
    ncclResult_t ar = ncclSuccess;
    ncclCommGetAsyncError((ncclComm_t)c->nccl_comm, &ar);
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if ((ar != ncclSuccess && ar != ncclInProgress) || dt > limit) {
      ncclCommAbort((ncclComm_t)c->nccl_comm);
      c->nccl_comm = nullptr;
      c->poisoned = true;
      return set_err(c, HHG_ERR_NCCL, ar != ncclSuccess && ar != ncclInProgress
                                          ? std::string("NCCL async error: ") + ncclGetErrorString(ar)
                                          : std::string("NCCL wait timed out"));
    }
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

void dist_destroy(Ctx* c) {
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  c->comm_stream = nullptr;
  if (c->nccl_comm) ncclCommDestroy((ncclComm_t)c->nccl_comm);
  c->nccl_comm = nullptr;
  if (c->h_stage) cudaFreeHost(c->h_stage);
  c->h_stage = nullptr;
}

// Pairwise exchange of byte ranges (buffers concatenated in rank order).
hhg_status dist_exchange_bytes(Ctx* c, const std::vector<int64_t>& sb, const void* send,
                               const std::vector<int64_t>& rb, void* recv, bool device, cudaStream_t stream) {
  if (!stream) stream = c->stream;
  const int nr = c->nranks;
  int64_t ts = 0, tr = 0;
  for (int p = 0; p < nr; ++p) ts += sb[p], tr += rb[p];
  if (c->transport == 1) {
    const char* s = (const char*)send;
    char* r = (char*)recv;
    void *ds = nullptr, *dr = nullptr;
    if (!device) {  // setup-time host data
      HHG_CK(c, cudaMalloc(&ds, std::max<int64_t>(ts, 1)));
      HHG_CK(c, cudaMalloc(&dr, std::max<int64_t>(tr, 1)));
      // stream-ordered before the sends (the ctx stream may be a non-blocking stream)
      HHG_CK(c, cudaMemcpyAsync(ds, send, ts, cudaMemcpyHostToDevice, stream));
      s = (const char*)ds;
      r = (char*)dr;
    }
    HHG_NCCL(c, ncclGroupStart());
    int64_t so = 0, ro = 0;
    for (int p = 0; p < nr; ++p) {
      if (sb[p]) HHG_NCCL(c, ncclSend(s + so, sb[p], ncclChar, p, (ncclComm_t)c->nccl_comm, stream));
      if (rb[p]) HHG_NCCL(c, ncclRecv(r + ro, rb[p], ncclChar, p, (ncclComm_t)c->nccl_comm, stream));
      so += sb[p];
      ro += rb[p];
    }
    HHG_NCCL(c, ncclGroupEnd());
    if (!device) {
      HHG_CK(c, cudaMemcpyAsync(recv, dr, tr, cudaMemcpyDeviceToHost, stream));
      { hhg_status st_sync__ = ctx_sync(c); if (st_sync__ != HHG_OK) return st_sync__; }
      cudaFree(ds);
      cudaFree(dr);
    }
    return HHG_OK;
  }
  if (c->transport == 2) {
    HostFn fn = (HostFn)c->host_fn;
    if (!device) {
      if (fn(c->host_user, nr, sb.data(), send, rb.data(), recv) != 0)
        return set_err(c, HHG_ERR_NCCL, "host transport failed");
      return HHG_OK;
    }
    const int64_t need = (ts + tr + 7) / 8;
    if (c->h_stage_n < need) {
      if (c->h_stage) cudaFreeHost(c->h_stage);
      HHG_CK(c, cudaMallocHost(&c->h_stage, need * 8));
      c->h_stage_n = need;
    }
    char* hs = (char*)c->h_stage;
    char* hr = hs + ts;
    HHG_CK(c, cudaMemcpyAsync(hs, send, ts, cudaMemcpyDeviceToHost, stream));
    HHG_CK(c, cudaStreamSynchronize(stream));
    if (fn(c->host_user, nr, sb.data(), hs, rb.data(), hr) != 0)
      return set_err(c, HHG_ERR_NCCL, "host transport failed");
    HHG_CK(c, cudaMemcpyAsync(recv, hr, tr, cudaMemcpyHostToDevice, stream));
    // the staging buffer is reused by the next exchange, possibly on another stream
    HHG_CK(c, cudaStreamSynchronize(stream));
    return HHG_OK;
  }
  return set_err(c, HHG_ERR_STATE, "no transport");
}

hhg_status dist_build_plan(Ctx* c, Level& lv, const std::vector<uint32_t>& recv_slot,
                           const std::vector<int64_t>& recv_gid, const std::vector<int32_t>& recv_rank,
                           const std::vector<std::pair<int64_t, uint32_t>>& serve) {
  const int nr = c->nranks;
  const int N = lv.N;
  const GidInfo& g = lv.gi;
  // group requests by owner rank (stable)
  std::vector<std::vector<size_t>> by(nr);
  for (size_t x = 0; x < recv_slot.size(); ++x) by[recv_rank[x]].push_back(x);
  lv.recv_cnt.assign(nr, 0);
  lv.h_recv_slot.clear();
  lv.h_recv_gid.clear();
  for (int p = 0; p < nr; ++p) {
    lv.recv_cnt[p] = (int64_t)by[p].size();
    for (size_t x : by[p]) {
      lv.h_recv_slot.push_back(recv_slot[x]);
      lv.h_recv_gid.push_back(recv_gid[x]);
    }
  }
  // counts: I tell every peer how many values I need from it
  std::vector<int64_t> one(nr, (int64_t)sizeof(int64_t));
  std::vector<int64_t> cnt_recv(nr, 0);
  hhg_status st = dist_exchange_bytes(c, one, lv.recv_cnt.data(), one, cnt_recv.data(), false, c->stream);
  if (st != HHG_OK) return st;
  lv.send_cnt = cnt_recv;
  std::vector<int64_t> sb(nr), rb(nr);
  int64_t nsend = 0;
  for (int p = 0; p < nr; ++p) {
    sb[p] = lv.recv_cnt[p] * 8;
    rb[p] = lv.send_cnt[p] * 8;
    nsend += lv.send_cnt[p];
  }
  std::vector<int64_t> asked(nsend);
  st = dist_exchange_bytes(c, sb, lv.h_recv_gid.data(), rb, asked.data(), false, c->stream);
  if (st != HHG_OK) return st;
  // resolve requested ids to this rank's authoritative slots
  std::vector<std::array<int, 3>> vinv(g.nvi);
  {
    int64_t x = 0;
    for (int k = 1; k < N; ++k)
      for (int j = 1; j < N - k; ++j)
        for (int i = 1; i < N - k - j; ++i) vinv[x++] = {i, j, k};
  }
  lv.h_send_slot.resize(nsend);
  lv.h_send_gid = asked;
  for (int64_t x = 0; x < nsend; ++x) {
    const int64_t gid = asked[x];
    int64_t slot = -1;
    if (gid >= g.base_v) {
      const int64_t gt = (gid - g.base_v) / g.nvi;
      const int64_t T = c->g2b[gt];
      if (T >= 0 && T < c->nt_local) {
        const auto& ijk = vinv[(gid - g.base_v) - gt * g.nvi];
        slot = T * lv.S + lattice_pos(N, ijk[0], ijk[1], ijk[2]);
      }
    } else {
      auto it = std::lower_bound(serve.begin(), serve.end(), std::make_pair(gid, (uint32_t)0));
      if (it != serve.end() && it->first == gid) slot = it->second;
    }
    if (slot < 0)
      return set_err(c, HHG_ERR_MESH, "exchange plan: rank " + std::to_string(c->rank) + " cannot serve node " +
                                           std::to_string(gid));
    lv.h_send_slot[x] = (uint32_t)slot;
  }
  lv.n_send = nsend;
  lv.n_recv = (int64_t)lv.h_recv_slot.size();
  // reverse grouping: one owner slot may be requested by several peers / copies
  std::vector<uint32_t> rptr, rslot, ridx(nsend);
  for (int64_t x = 0; x < nsend; ++x) ridx[x] = (uint32_t)x;
  std::stable_sort(ridx.begin(), ridx.end(),
                   [&](uint32_t a, uint32_t b) { return lv.h_send_slot[a] < lv.h_send_slot[b]; });
  for (int64_t x = 0; x < nsend; ++x) {
    if (x == 0 || lv.h_send_slot[ridx[x]] != lv.h_send_slot[ridx[x - 1]]) {
      rptr.push_back((uint32_t)x);
      rslot.push_back(lv.h_send_slot[ridx[x]]);
    }
  }
  rptr.push_back((uint32_t)nsend);
  lv.n_rsum = (int64_t)rslot.size();
  if (c->host_only) return HHG_OK;
  HHG_CK(c, cudaMalloc(&lv.d_rsum_ptr, rptr.size() * 4));
  HHG_CK(c, cudaMalloc(&lv.d_rsum_slot, std::max<int64_t>(lv.n_rsum, 1) * 4));
  HHG_CK(c, cudaMalloc(&lv.d_rsum_idx, std::max<int64_t>(nsend, 1) * 4));
  HHG_CK(c, cudaMemcpy(lv.d_rsum_ptr, rptr.data(), rptr.size() * 4, cudaMemcpyHostToDevice));
  if (lv.n_rsum) HHG_CK(c, cudaMemcpy(lv.d_rsum_slot, rslot.data(), lv.n_rsum * 4, cudaMemcpyHostToDevice));
  if (nsend) HHG_CK(c, cudaMemcpy(lv.d_rsum_idx, ridx.data(), nsend * 4, cudaMemcpyHostToDevice));
  HHG_CK(c, cudaMalloc(&lv.d_send_slot, std::max<int64_t>(lv.n_send, 1) * 4));
  HHG_CK(c, cudaMalloc(&lv.d_recv_slot, std::max<int64_t>(lv.n_recv, 1) * 4));
  HHG_CK(c, cudaMalloc(&lv.d_sendbuf, std::max<int64_t>(lv.n_send, 1) * 8));
  HHG_CK(c, cudaMalloc(&lv.d_recvbuf, std::max<int64_t>(lv.n_recv, 1) * 8));
  if (lv.n_send)
    HHG_CK(c, cudaMemcpy(lv.d_send_slot, lv.h_send_slot.data(), lv.n_send * 4, cudaMemcpyHostToDevice));
  if (lv.n_recv)
    HHG_CK(c, cudaMemcpy(lv.d_recv_slot, lv.h_recv_slot.data(), lv.n_recv * 4, cudaMemcpyHostToDevice));
  return HHG_OK;
}

__global__ void k_pack(int64_t n, const uint32_t* __restrict__ slot, const double* __restrict__ v,
                       double* __restrict__ buf) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) buf[t] = v[slot[t]];
}

__global__ void k_unpack(int64_t n, const uint32_t* __restrict__ slot, const double* __restrict__ buf,
                         double* __restrict__ v) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) v[slot[t]] = buf[t];
}

hhg_status dist_sync(Ctx* c, Level& lv, double* v, cudaStream_t stream) {
  if (c->nranks == 1) return HHG_OK;
  if (!stream) stream = c->stream;
  ProfScope ps(c, 3);
  if (lv.n_send) {
    k_pack<<<(unsigned)((lv.n_send + 255) / 256), 256, 0, stream>>>(lv.n_send, lv.d_send_slot, v, lv.d_sendbuf);
    HHG_LAUNCHED(c);
  }
  std::vector<int64_t> sb(c->nranks), rb(c->nranks);
  for (int p = 0; p < c->nranks; ++p) {
    sb[p] = lv.send_cnt[p] * 8;
    rb[p] = lv.recv_cnt[p] * 8;
  }
  hhg_status st = dist_exchange_bytes(c, sb, lv.d_sendbuf, rb, lv.d_recvbuf, true, stream);
  if (st != HHG_OK) return st;
  if (lv.n_recv) {
    k_unpack<<<(unsigned)((lv.n_recv + 255) / 256), 256, 0, stream>>>(lv.n_recv, lv.d_recv_slot, lv.d_recvbuf, v);
    HHG_LAUNCHED(c);
  }
  return HHG_OK;
}

// Ghost exchange of v overlapped with compute: the exchange runs
// on the ctx's communication stream after everything enqueued so far on the
// ctx stream (the values it sends are final), while `interior` -- work that
// neither writes a sent value nor reads / writes a received slot -- is
// enqueued on the ctx stream; the ctx stream then waits for the exchange.
hhg_status dist_sync_overlapped(Ctx* c, Level& lv, double* v, const std::function<hhg_status()>& interior) {
  if (c->nranks == 1) return interior();
  if (!c->comm_stream) {
    HHG_CK(c, cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    HHG_CK(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    HHG_CK(c, cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  }
  HHG_CK(c, cudaEventRecord(c->ev_fork, c->stream));
  HHG_CK(c, cudaStreamWaitEvent(c->comm_stream, c->ev_fork, 0));
  // the interior work is enqueued first: with the host transport the exchange
  // blocks this thread, and the GPU must already have the interior kernels
  hhg_status st = interior();
  if (st != HHG_OK) return st;
  if ((st = dist_sync(c, lv, v, c->comm_stream)) != HHG_OK) return st;
  HHG_CK(c, cudaEventRecord(c->ev_join, c->comm_stream));
  HHG_CK(c, cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  return HHG_OK;
}

// owner slot += the copies' partial values (fixed order: deterministic)
__global__ void k_unpack_sum(int64_t n, const uint32_t* __restrict__ ptr, const uint32_t* __restrict__ slot,
                             const uint32_t* __restrict__ idx, const double* __restrict__ buf,
                             double* __restrict__ v) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  double s = 0.0;
  for (uint32_t e = ptr[t]; e < ptr[t + 1]; ++e) s += buf[idx[e]];
  v[slot[t]] += s;
}

// Reverse of dist_sync: every mirrored slot sends its value to the owner,
// which adds them into its authoritative slot (restriction partial sums,
// PAPER.md:852-860 R = P^T across a rank boundary).  The mirrored slots keep
// their values; callers re-sync after summing the owner's local copies.
hhg_status dist_sum_to_owner(Ctx* c, Level& lv, double* v) {
  if (c->nranks == 1) return HHG_OK;
  ProfScope ps(c, 3);
  if (lv.n_recv) {
    k_pack<<<(unsigned)((lv.n_recv + 255) / 256), 256, 0, c->stream>>>(lv.n_recv, lv.d_recv_slot, v, lv.d_recvbuf);
    HHG_LAUNCHED(c);
  }
  std::vector<int64_t> sb(c->nranks), rb(c->nranks);
  for (int p = 0; p < c->nranks; ++p) {
    sb[p] = lv.recv_cnt[p] * 8;
    rb[p] = lv.send_cnt[p] * 8;
  }
  hhg_status st = dist_exchange_bytes(c, sb, lv.d_recvbuf, rb, lv.d_sendbuf, true, c->stream);
  if (st != HHG_OK) return st;
  if (lv.n_rsum) {
    k_unpack_sum<<<(unsigned)((lv.n_rsum + 255) / 256), 256, 0, c->stream>>>(lv.n_rsum, lv.d_rsum_ptr, lv.d_rsum_slot,
                                                                             lv.d_rsum_idx, lv.d_sendbuf, v);
    HHG_LAUNCHED(c);
  }
  return HHG_OK;
}

__global__ void k_sum_ranks(int nr, const double* __restrict__ parts, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int p = 0; p < nr; ++p) s += parts[p];  // rank order: identical on every rank
    out[0] = s;
  }
}

// *d_scalar <- sum over ranks (deterministic, rank order)
hhg_status dist_allreduce_sum(Ctx* c, double* d_scalar) {
  if (c->nranks == 1) return HHG_OK;
  const int nr = c->nranks;
  double* buf = nullptr;
  HHG_CK(c, cudaMallocAsync((void**)&buf, 2 * nr * sizeof(double), c->stream));
  for (int p = 0; p < nr; ++p)
    HHG_CK(c, cudaMemcpyAsync(buf + p, d_scalar, 8, cudaMemcpyDeviceToDevice, c->stream));
  std::vector<int64_t> sb(nr, 8), rb(nr, 8);
  sb[c->rank] = 0;
  rb[c->rank] = 0;
  // own contribution goes straight to its rank slot of the receive half
  HHG_CK(c, cudaMemcpyAsync(buf + nr + c->rank, d_scalar, 8, cudaMemcpyDeviceToDevice, c->stream));
  // exchange: send buf[0..nr) (skipping self), receive into buf[nr..2nr) (skipping self)
  {
    std::vector<int64_t> sbc(nr), rbc(nr);
    for (int p = 0; p < nr; ++p) sbc[p] = sb[p], rbc[p] = rb[p];
    // pack contiguous send / recv views without the self slot
    double* sendv = buf;                 // nr entries, self entry unused (0 bytes)
    double* recvv = nullptr;
    HHG_CK(c, cudaMallocAsync((void**)&recvv, nr * sizeof(double), c->stream));
    hhg_status st = dist_exchange_bytes(c, sbc, sendv, rbc, recvv, true, c->stream);
    if (st != HHG_OK) return st;
    // recvv holds the peers' values in rank order (self skipped): scatter into buf[nr..]
    int q = 0;
    for (int p = 0; p < nr; ++p) {
      if (p == c->rank) continue;
      HHG_CK(c, cudaMemcpyAsync(buf + nr + p, recvv + q, 8, cudaMemcpyDeviceToDevice, c->stream));
      ++q;
    }
    cudaFreeAsync(recvv, c->stream);
  }
  k_sum_ranks<<<1, 32, 0, c->stream>>>(nr, buf + nr, d_scalar);
  HHG_LAUNCHED(c);
  cudaFreeAsync(buf, c->stream);
  return HHG_OK;
}

__global__ void k_sum_vec_ranks(int nr, int rank, int64_t n, const double* __restrict__ recv,
                                double* __restrict__ v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  int q = 0;
  for (int p = 0; p < nr; ++p) s += (p == rank) ? v[i] : recv[(int64_t)(q++) * n + i];  // rank order
  v[i] = s;
}

// d_vec[0..n) <- elementwise sum over ranks, identical on every rank (NCCL
// all-reduce; host transport: all-gather + rank-order sum).  Used for vectors
// whose entries are nonzero on exactly one rank, where every order is exact.
hhg_status dist_allreduce_vec(Ctx* c, double* d_vec, int64_t n) {
  if (c->nranks == 1 || n == 0) return HHG_OK;
  const int nr = c->nranks;
  if (c->transport == 1) {
    HHG_NCCL(c, ncclAllReduce(d_vec, d_vec, (size_t)n, ncclDouble, ncclSum, (ncclComm_t)c->nccl_comm, c->stream));
    return HHG_OK;
  }
  double *sendv = nullptr, *recvv = nullptr;
  HHG_CK(c, cudaMallocAsync((void**)&sendv, (size_t)(nr - 1) * n * sizeof(double), c->stream));
  HHG_CK(c, cudaMallocAsync((void**)&recvv, (size_t)(nr - 1) * n * sizeof(double), c->stream));
  for (int q = 0; q < nr - 1; ++q)
    HHG_CK(c, cudaMemcpyAsync(sendv + (int64_t)q * n, d_vec, n * sizeof(double), cudaMemcpyDeviceToDevice,
                              c->stream));
  std::vector<int64_t> sb(nr, n * 8), rb(nr, n * 8);
  sb[c->rank] = 0;
  rb[c->rank] = 0;
  hhg_status st = dist_exchange_bytes(c, sb, sendv, rb, recvv, true, c->stream);
  if (st != HHG_OK) return st;
  k_sum_vec_ranks<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(nr, c->rank, n, recvv, d_vec);
  HHG_LAUNCHED(c);
  cudaFreeAsync(sendv, c->stream);
  cudaFreeAsync(recvv, c->stream);
  return HHG_OK;
}

}  // namespace hhg

using namespace hhg;

extern "C" hhg_status hhg_nccl_unique_id(void* out128) {
  if (!out128) return HHG_ERR_INVALID;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return HHG_ERR_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
  std::memcpy(out128, &id, sizeof(id));
  return HHG_OK;
}

extern "C" hhg_status hhg_set_host_transport(hhg_host_exchange_fn fn, void* user, int host_only) {
  g_host_fn = (HostFn)fn;
  g_host_user = user;
  g_host_only = host_only;
  return HHG_OK;
}

extern "C" hhg_status hhg_plan_info(hhg_ctx ctx, int L, int64_t* info) {
  Ctx* c = (Ctx*)ctx;
  if (!c || L < 2 || L > c->L_max || !info) return HHG_ERR_INVALID;
  const Level& lv = c->levels[L];
  info[0] = lv.n_owned;
  info[1] = lv.n_send;
  info[2] = lv.n_recv;
  info[3] = c->nt_local;
  info[4] = c->nt_blocks;
  return HHG_OK;
}

// Runs the exchange plan on canonical node ids through the transport and counts
// received ids that differ from the ids this rank expected (0 = plan consistent).
extern "C" hhg_status hhg_plan_check(hhg_ctx ctx, int L, int64_t* mismatches) {
  Ctx* c = (Ctx*)ctx;
  if (!c || L < 2 || L > c->L_max || !mismatches) return HHG_ERR_INVALID;
  Level& lv = c->levels[L];
  if (c->nranks == 1) {
    *mismatches = 0;
    return HHG_OK;
  }
  std::vector<int64_t> sb(c->nranks), rb(c->nranks);
  for (int p = 0; p < c->nranks; ++p) {
    sb[p] = lv.send_cnt[p] * 8;
    rb[p] = lv.recv_cnt[p] * 8;
  }
  std::vector<int64_t> got(lv.n_recv);
  hhg_status st = dist_exchange_bytes(c, sb, lv.h_send_gid.data(), rb, got.data(), false, c->stream);
  if (st != HHG_OK) return st;
  int64_t bad = 0;
  for (int64_t x = 0; x < lv.n_recv; ++x) bad += got[x] != lv.h_recv_gid[x];
  *mismatches = bad;
  return HHG_OK;
}
