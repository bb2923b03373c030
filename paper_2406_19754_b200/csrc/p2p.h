// p2p.h — NVLink peer-memory exchanges (see p2p.cu).
#pragma once
#include <map>
#include <vector>

#include "kernels.h"
#include "psc_internal.h"

namespace psc {

struct P2PBufSpec {  // a halo-bearing vector in the arena, exchanged at `level`
  double* local;
  int level;
};
struct P2PGatherSpec {  // an all-gather target in the arena; my block starts at local + my_block
  double* local;
  int64_t my_block;
};
struct P2PBufDev {
  int level = -1;
  double** d_dst = nullptr;  // [R] device pointers into peer memory
};
struct P2PLevel {
  bool any = false;
  int64_t max_send = 0;
  int32_t* d_nbr = nullptr;
  int64_t* d_soff = nullptr;
  // fused push: for each owned row, its sends (peer, slot in the peer's block)
  int32_t* d_iptr = nullptr;
  uint8_t* d_sslice = nullptr;
  int32_t* d_iq = nullptr;
  int32_t* d_ipos = nullptr;
};
struct P2P {
  bool on = false;
  char* arena = nullptr;  // this rank's IPC-shared allocation (owned by the hierarchy)
  std::vector<char*> peer_arena;
  uint64_t* flags = nullptr;  // [R] in the arena
  uint64_t** d_pflag = nullptr;
  uint64_t* d_gen = nullptr;
  unsigned int* d_ticket = nullptr;
  unsigned int* d_ticket_push = nullptr;  // fused pushes (producer row kernels)
  int32_t* d_all = nullptr;
  std::vector<P2PLevel> levels;
  std::map<const double*, P2PBufDev> bufs;
  std::map<const double*, P2PBufDev> gathers;
};

// collective; P.arena must be set and the flags region zeroed
void p2p_setup(psc_ctx* ctx, P2P& P, const std::vector<P2PBufSpec>& halo_bufs,
               const std::vector<P2PGatherSpec>& gathers, const std::vector<psc_desc*>& level_desc,
               int64_t flags_off);
void p2p_free(psc_ctx* ctx, P2P& P);
// collective: the minimum of v over all ranks (NCCL all-reduce on ctx's stream)
int allreduce_min(psc_ctx* ctx, int v);
// false: not handled (caller falls back to NCCL)
bool p2p_halo(psc_ctx* ctx, P2P& P, psc_desc* d, const double* x, cudaStream_t s);
// Fused push of a row kernel's output y (a registered halo-bearing vector of the row
// space d) / wait in the kernel that next reads x's halo.  false: not possible (the
// caller exchanges with p2p_halo).  See PushSpec / WaitSpec (kernels.h).
bool p2p_push_spec(psc_ctx* ctx, P2P& P, psc_desc* d, const double* y, PushSpec& ps);
bool p2p_wait_spec(psc_ctx* ctx, P2P& P, const double* x, WaitSpec& ws);
bool p2p_allgather(psc_ctx* ctx, P2P& P, const double* src, int64_t n, const double* dst_base_local,
                   cudaStream_t s);

}  // namespace psc
