// p2p.cu — NVLink peer-memory halo exchange and all-gathers (one node, one process per GPU).
//
// The halo exchange before every sweep / SpMV ("neighbourhood data
// communications"; P:157-158 GPU-side packing) and the per-rank scalar
// all-gathers of the CG reductions are done by ONE kernel each, writing
// directly into the peers' memory over NVLink/NVSwitch:
//   pack x[send_idx] -> st.global into the peer's halo slots (CUDA IPC mapping)
//   -> __threadfence_system per CTA -> last CTA: st.release.sys of a per-pair
//   generation counter into each neighbour's flag word, then ld.acquire.sys spin
//   until every neighbour's counter for this exchange has arrived.
// Generation counters live on the device, so the exchange replays correctly
// inside the captured iteration graph.  Every exchange is a mutual barrier among
// the (symmetric) neighbour set of its level, which also orders a peer's next
// write into a buffer after this rank's last read of it.  NCCL remains the
// fallback (PSC_NO_P2P=1, two ranks on one device, or IPC/P2P unavailable).
#include <cstring>

#include "kernels.h"
#include "p2p.h"

namespace psc {

static __device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
static __device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

struct PushArgs {
  const double* x;        // source (owned part)
  const int32_t* idx;     // gather indices into x (halo); nullptr: x[k] (all-gather)
  const int64_t* soff;    // [R+1] per-peer offsets into idx (halo); nullptr: n entries for every peer
  int64_t n;              // entries per peer when soff == nullptr
  double* const* dst;     // [R] destination in peer p's memory (nullptr: nothing for p)
  const int32_t* nbr;     // [R] 1 = exchange partner (signal + wait)
  uint64_t* const* pflag; // [R] &flags_p[me] (peer memory)
  const uint64_t* myflag; // [R] my flag words, written by the peers
  uint64_t* gen;          // [2R] sgen[p], rgen[p]
  unsigned int* ticket;
  int R;
  uint64_t timeout_ns;  // bound of the wait for a peer's flag (then __trap: a launch error, not a hang)
  int fence;            // 0: fence.sc.sys per CTA; 1: fence.acq_rel.sys (PSC_P2P_FENCE)
};

static __device__ __forceinline__ void fence_sys(int mode) {
  if (mode == 1) asm volatile("fence.acq_rel.sys;" ::: "memory");
  else __threadfence_system();
}

static __device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(256) p2p_push_kernel(PushArgs a) {
  const int p = blockIdx.y;
  double* d = a.dst[p];
  if (d) {
    const int64_t b = a.soff ? a.soff[p] : 0;
    const int64_t n = a.soff ? a.soff[p + 1] - b : a.n;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
      d[k] = a.idx ? a.x[a.idx[b + k]] : a.x[k];
  }
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_sys(a.fence);
    const unsigned int t = atomicAdd(a.ticket, 1u);
    last = (t == gridDim.x * gridDim.y - 1);
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  fence_sys(a.fence);
  for (int q = 0; q < a.R; ++q)
    if (a.nbr[q]) st_release_sys(a.pflag[q], ++a.gen[q]);
  // wait until every neighbour has signalled as often as this rank has (the signal
  // counts of a pair advance in the same collective order on both sides; fused
  // pushes in row kernels signal without a standalone exchange, PushSpec)
  const uint64_t t0 = globaltimer();
  for (int q = 0; q < a.R; ++q)
    if (a.nbr[q]) {
      const uint64_t target = a.gen[q];
      while (ld_acquire_sys(a.myflag + q) < target) {
        // a peer that never signals (crashed, or left the collective order) must not
        // hang this GPU: after timeout_ns the kernel traps and the host call returns
        // PSC_ERR_CUDA (the library then aborts the NCCL communicator)
        if (globaltimer() - t0 > a.timeout_ns) __trap();
      }
    }
  __threadfence();
  *a.ticket = 0u;
}

// PSC_SPIN_TIMEOUT_S: seconds a rank waits for a neighbour's flag (default 300: ranks can
// legitimately drift apart by tens of seconds on large set-ups, e.g. 512^3 over 4 GPUs
// with host-side inputs, where a 30 s bound tripped)
static uint64_t spin_timeout_ns() {
  static const uint64_t tmo =
      (uint64_t)(1e9 * (getenv("PSC_SPIN_TIMEOUT_S") ? atof(getenv("PSC_SPIN_TIMEOUT_S")) : 300.0));
  return tmo;
}

static void push(psc_ctx* ctx, P2P& P, const double* x, const int32_t* idx, const int64_t* soff, int64_t n,
                 int64_t max_per_peer, double* const* dst, const int32_t* nbr, cudaStream_t s) {
  const uint64_t tmo = spin_timeout_ns();
  static const int fence = getenv("PSC_P2P_FENCE") ? atoi(getenv("PSC_P2P_FENCE")) : 0;
  static const int64_t bxmax = getenv("PSC_P2P_BX") ? std::max(1, atoi(getenv("PSC_P2P_BX"))) : 64;
  static const int64_t per_cta = getenv("PSC_P2P_PER_CTA") ? std::max(32, atoi(getenv("PSC_P2P_PER_CTA"))) : 256;
  PushArgs a{x, idx, soff, n, dst, nbr, P.d_pflag, P.flags, P.d_gen, P.d_ticket, ctx->nranks, tmo, fence};
  KtScope kts(ctx, s, idx ? "p2p_halo" : "p2p_allgather", 0.0, 0.0);
  const int64_t bx = std::max<int64_t>(1, std::min<int64_t>((max_per_peer + per_cta - 1) / per_cta, bxmax));
  p2p_push_kernel<<<dim3((unsigned)bx, (unsigned)ctx->nranks), 256, 0, s>>>(a);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
  ctx->collectives++;
}

bool p2p_halo(psc_ctx* ctx, P2P& P, psc_desc* d, const double* x, cudaStream_t s) {
  if (!P.on) return false;
  auto it = P.bufs.find(x);
  if (it == P.bufs.end()) return false;
  const P2PLevel& L = P.levels[it->second.level];
  if (!L.any) return true;  // no neighbour at this level: nothing to exchange
  push(ctx, P, x, d->d_send_idx, L.d_soff, 0, L.max_send, it->second.d_dst, L.d_nbr, s);
  return true;
}

bool p2p_push_spec(psc_ctx* ctx, P2P& P, psc_desc* d, const double* y, PushSpec& ps) {
  ps = PushSpec();
  if (!P.on) return false;
  auto it = P.bufs.find(y);
  if (it == P.bufs.end()) return false;
  const P2PLevel& L = P.levels[it->second.level];
  if (!L.any || !L.d_iptr || d->n_own + d->n_halo() <= 0) return false;
  ps.on = 1;
  ps.R = ctx->nranks;
  ps.sslice = L.d_sslice;
  ps.iptr = L.d_iptr;
  ps.iq = L.d_iq;
  ps.ipos = L.d_ipos;
  ps.dst = it->second.d_dst;
  ps.nbr = L.d_nbr;
  ps.pflag = P.d_pflag;
  ps.gen = P.d_gen;
  ps.ticket = P.d_ticket_push;
  ctx->collectives++;
  return true;
}

bool p2p_wait_spec(psc_ctx* ctx, P2P& P, const double* x, WaitSpec& ws) {
  ws = WaitSpec();
  if (!P.on) return false;
  auto it = P.bufs.find(x);
  if (it == P.bufs.end()) return false;
  const P2PLevel& L = P.levels[it->second.level];
  ws.on = L.any ? 1 : 0;
  ws.R = ctx->nranks;
  ws.nbr = L.d_nbr;
  ws.myflag = P.flags;
  ws.gen = P.d_gen;
  ws.timeout_ns = spin_timeout_ns();
  return true;
}

bool p2p_allgather(psc_ctx* ctx, P2P& P, const double* src, int64_t n, const double* dst_base_local,
                   cudaStream_t s) {
  if (!P.on) return false;
  auto it = P.gathers.find(dst_base_local);
  if (it == P.gathers.end()) return false;
  push(ctx, P, src, nullptr, nullptr, n, n, it->second.d_dst, P.d_all, s);
  return true;
}

// ---------------------------------------------------------------- set-up
static void allgather_bytes(psc_ctx* ctx, const void* mine, void* all, size_t bytes) {
  const int R = ctx->nranks;
  char* d = dalloc<char>(bytes * (R + 1));
  PSC_CUDA(cudaMemcpy(d + bytes * R, mine, bytes, cudaMemcpyHostToDevice));
  PSC_NCCL(ncclAllGather(d + bytes * R, d, bytes, ncclChar, ctx->comm, ctx->stream));
  PSC_CUDA(cudaMemcpyAsync(all, d, bytes * R, cudaMemcpyDeviceToHost, ctx->stream));
  PSC_CUDA(cudaStreamSynchronize(ctx->stream));
  dfree(d);
}

int allreduce_min(psc_ctx* ctx, int v) {
  int* d = dalloc<int>(1);
  PSC_CUDA(cudaMemcpy(d, &v, sizeof(int), cudaMemcpyHostToDevice));
  PSC_NCCL(ncclAllReduce(d, d, 1, ncclInt, ncclMin, ctx->comm, ctx->stream));
  PSC_CUDA(cudaMemcpyAsync(&v, d, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  PSC_CUDA(cudaStreamSynchronize(ctx->stream));
  dfree(d);
  return v;
}

void p2p_setup(psc_ctx* ctx, P2P& P, const std::vector<P2PBufSpec>& halo_bufs,
               const std::vector<P2PGatherSpec>& gathers, const std::vector<psc_desc*>& level_desc,
               int64_t flags_off) {
  const int R = ctx->nranks, me = ctx->rank;
  P.on = false;
  int ok = (R > 1 && !getenv("PSC_NO_P2P") && P.arena) ? 1 : 0;
  // distinct physical devices (P2P between two ranks of one GPU would need no
  // NVLink but the spin-waits must never share a device)
  char bus[64] = {0};
  PSC_CUDA(cudaDeviceGetPCIBusId(bus, sizeof(bus), ctx->device));
  std::vector<char> allbus(64 * R);
  allgather_bytes(ctx, bus, allbus.data(), 64);
  for (int p = 0; p < R; ++p)
    if (p != me && std::strncmp(&allbus[64 * p], bus, 64) == 0) ok = 0;
  cudaIpcMemHandle_t hdl;
  std::memset(&hdl, 0, sizeof(hdl));
  if (ok && cudaIpcGetMemHandle(&hdl, P.arena) != cudaSuccess) {
    cudaGetLastError();
    ok = 0;
  }
  std::vector<cudaIpcMemHandle_t> all(R);
  allgather_bytes(ctx, &hdl, all.data(), sizeof(hdl));
  P.peer_arena.assign(R, nullptr);
  P.peer_arena[me] = P.arena;
  for (int p = 0; p < R && ok; ++p) {
    if (p == me) continue;
    void* ptr = nullptr;
    if (cudaIpcOpenMemHandle(&ptr, all[p], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ok = 0;
      break;
    }
    P.peer_arena[p] = static_cast<char*>(ptr);
  }
  ok = allreduce_min(ctx, ok);  // every rank agrees (also a barrier after the flags were zeroed)
  if (!ok) {
    for (int p = 0; p < R; ++p)
      if (p != me && P.peer_arena[p]) cudaIpcCloseMemHandle(P.peer_arena[p]);
    P.peer_arena.clear();
    return;
  }
  // buffer offsets inside every rank's arena (same enumeration on all ranks)
  const size_t nb = halo_bufs.size() + gathers.size() + 1;
  std::vector<int64_t> myoff(nb);
  for (size_t b = 0; b < halo_bufs.size(); ++b) myoff[b] = (char*)halo_bufs[b].local - P.arena;
  for (size_t g = 0; g < gathers.size(); ++g) myoff[halo_bufs.size() + g] = (char*)gathers[g].local - P.arena;
  myoff[nb - 1] = flags_off;
  std::vector<int64_t> off((size_t)R * nb);
  allgather_bytes(ctx, myoff.data(), off.data(), nb * sizeof(int64_t));
  // per level: where my block starts in every peer's halo (peer's roff[me])
  const int L = (int)level_desc.size();
  std::vector<int64_t> myroff((size_t)L * (R + 1));
  for (int l = 0; l < L; ++l)
    for (int p = 0; p <= R; ++p) myroff[(size_t)l * (R + 1) + p] = level_desc[l]->roff[p];
  std::vector<int64_t> roff((size_t)R * L * (R + 1));
  allgather_bytes(ctx, myroff.data(), roff.data(), myroff.size() * sizeof(int64_t));
  P.levels.assign(L, P2PLevel());
  for (int l = 0; l < L; ++l) {
    psc_desc* d = level_desc[l];
    P2PLevel& Lv = P.levels[l];
    std::vector<int32_t> nbr(R, 0);
    for (int p = 0; p < R; ++p) {
      nbr[p] = (p != me && (d->scount[p] > 0 || d->rcount[p] > 0)) ? 1 : 0;
      Lv.any |= nbr[p] != 0;
      Lv.max_send = std::max<int64_t>(Lv.max_send, d->scount[p]);
    }
    Lv.d_nbr = dalloc<int32_t>(R);
    Lv.d_soff = dalloc<int64_t>(R + 1);
    PSC_CUDA(cudaMemcpy(Lv.d_nbr, nbr.data(), sizeof(int32_t) * R, cudaMemcpyHostToDevice));
    PSC_CUDA(cudaMemcpy(Lv.d_soff, d->soff.data(), sizeof(int64_t) * (R + 1), cudaMemcpyHostToDevice));
    // fused push: owned row -> (peer, position in my block of that peer's halo)
    if (d->n_send > 0) {
      std::vector<int32_t> sidx(d->n_send);
      PSC_CUDA(cudaMemcpy(sidx.data(), d->d_send_idx, sizeof(int32_t) * d->n_send, cudaMemcpyDeviceToHost));
      std::vector<int32_t> iptr(d->n_own + 1, 0), iq(d->n_send), ipos(d->n_send);
      for (int64_t k = 0; k < d->n_send; ++k) iptr[sidx[k] + 1]++;
      for (int64_t i = 0; i < d->n_own; ++i) iptr[i + 1] += iptr[i];
      std::vector<int32_t> fill(iptr.begin(), iptr.end() - 1);
      for (int p = 0; p < R; ++p)
        for (int64_t k = d->soff[p]; k < d->soff[p + 1]; ++k) {
          const int32_t o = fill[sidx[k]]++;
          iq[o] = p;
          ipos[o] = (int32_t)(k - d->soff[p]);
        }
      std::vector<uint8_t> ss((d->n_own + 31) / 32, 0);
      for (int64_t i = 0; i < d->n_own; ++i)
        if (iptr[i + 1] > iptr[i]) ss[i >> 5] = 1;
      Lv.d_sslice = dalloc<uint8_t>(ss.size());
      PSC_CUDA(cudaMemcpy(Lv.d_sslice, ss.data(), ss.size(), cudaMemcpyHostToDevice));
      Lv.d_iptr = dalloc<int32_t>(d->n_own + 1);
      Lv.d_iq = dalloc<int32_t>(d->n_send);
      Lv.d_ipos = dalloc<int32_t>(d->n_send);
      PSC_CUDA(cudaMemcpy(Lv.d_iptr, iptr.data(), sizeof(int32_t) * (d->n_own + 1), cudaMemcpyHostToDevice));
      PSC_CUDA(cudaMemcpy(Lv.d_iq, iq.data(), sizeof(int32_t) * d->n_send, cudaMemcpyHostToDevice));
      PSC_CUDA(cudaMemcpy(Lv.d_ipos, ipos.data(), sizeof(int32_t) * d->n_send, cudaMemcpyHostToDevice));
    }
  }
  for (size_t b = 0; b < halo_bufs.size(); ++b) {
    const int l = halo_bufs[b].level;
    psc_desc* d = level_desc[l];
    std::vector<double*> dst(R, nullptr);
    for (int p = 0; p < R; ++p) {
      if (p == me || d->scount[p] == 0) continue;
      const int64_t n_own_p = d->row_start[p + 1] - d->row_start[p];
      const int64_t roff_p_me = roff[((size_t)p * L + l) * (R + 1) + me];
      dst[p] = reinterpret_cast<double*>(P.peer_arena[p] + off[(size_t)p * nb + b]) + n_own_p + roff_p_me;
    }
    P2PBufDev bd;
    bd.level = l;
    bd.d_dst = dalloc<double*>(R);
    PSC_CUDA(cudaMemcpy(bd.d_dst, dst.data(), sizeof(double*) * R, cudaMemcpyHostToDevice));
    P.bufs[halo_bufs[b].local] = bd;
  }
  // all-gathers: my block goes to gathers[g].local + my block offset in every rank (me included)
  std::vector<int32_t> allnbr(R, 1);
  allnbr[me] = 0;
  P.d_all = dalloc<int32_t>(R);
  PSC_CUDA(cudaMemcpy(P.d_all, allnbr.data(), sizeof(int32_t) * R, cudaMemcpyHostToDevice));
  for (size_t g = 0; g < gathers.size(); ++g) {
    std::vector<double*> dst(R, nullptr);
    for (int p = 0; p < R; ++p)
      dst[p] = reinterpret_cast<double*>(P.peer_arena[p] + off[(size_t)p * nb + halo_bufs.size() + g]) +
               gathers[g].my_block;
    P2PBufDev bd;
    bd.level = -1;
    bd.d_dst = dalloc<double*>(R);
    PSC_CUDA(cudaMemcpy(bd.d_dst, dst.data(), sizeof(double*) * R, cudaMemcpyHostToDevice));
    P.gathers[gathers[g].local] = bd;
  }
  // flags: mine in my arena; peer_flag[p] = &flags_p[me]
  P.flags = reinterpret_cast<uint64_t*>(P.arena + flags_off);
  std::vector<uint64_t*> pf(R, nullptr);
  for (int p = 0; p < R; ++p)
    if (p != me) pf[p] = reinterpret_cast<uint64_t*>(P.peer_arena[p] + off[(size_t)p * nb + nb - 1]) + me;
  P.d_pflag = dalloc<uint64_t*>(R);
  PSC_CUDA(cudaMemcpy(P.d_pflag, pf.data(), sizeof(uint64_t*) * R, cudaMemcpyHostToDevice));
  P.d_gen = dalloc<uint64_t>(2 * R);
  PSC_CUDA(cudaMemset(P.d_gen, 0, sizeof(uint64_t) * 2 * R));
  P.d_ticket = dalloc<unsigned int>(1);
  PSC_CUDA(cudaMemset(P.d_ticket, 0, sizeof(unsigned int)));
  P.d_ticket_push = dalloc<unsigned int>(1);
  PSC_CUDA(cudaMemset(P.d_ticket_push, 0, sizeof(unsigned int)));
  PSC_CUDA(cudaDeviceSynchronize());
  allreduce_min(ctx, 1);  // nobody signals before everybody is set up
  P.on = true;
}

void p2p_free(psc_ctx* ctx, P2P& P) {
  for (size_t p = 0; p < P.peer_arena.size(); ++p)
    if ((int)p != ctx->rank && P.peer_arena[p]) cudaIpcCloseMemHandle(P.peer_arena[p]);
  for (auto& kv : P.bufs) dfree(kv.second.d_dst);
  for (auto& kv : P.gathers) dfree(kv.second.d_dst);
  for (auto& Lv : P.levels) {
    dfree(Lv.d_nbr);
    dfree(Lv.d_soff);
    dfree(Lv.d_iptr);
    dfree(Lv.d_sslice);
    dfree(Lv.d_iq);
    dfree(Lv.d_ipos);
  }
  dfree(P.d_all);
  dfree(P.d_pflag);
  dfree(P.d_gen);
  dfree(P.d_ticket);
  dfree(P.d_ticket_push);
  P = P2P();
}

}  // namespace psc
