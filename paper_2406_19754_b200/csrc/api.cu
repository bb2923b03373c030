// api.cu — context, descriptors (index spaces + halo plans) and matrices of
// libpsc.so.  PSBLAS lifecycle of PAPER.md P:79-107 (Sec. 2.1).
#include <algorithm>
#include <cstring>

#include "kernels.h"

using namespace psc;

namespace {

thread_local std::string g_err;  // last error without a context (psc_init failures)

int fail(psc_ctx* ctx, const Error& e) {
  if (ctx) ctx->err = e.what();
  g_err = e.what();
  // A device fault (e.g. a peer-flag wait that timed out and trapped, p2p.cu) or an
  // NCCL failure leaves the other ranks inside a collective: abort the communicator
  // so their NCCL calls return an error instead of hanging.  Later collective calls
  // on this context fail with PSC_ERR_STATE.
  if (ctx && ctx->comm && ctx->nranks > 1 && (e.code == PSC_ERR_CUDA || e.code == PSC_ERR_NCCL)) {
    ncclCommAbort(ctx->comm);
    ctx->comm = nullptr;
  }
  return e.code;
}
int fail(psc_ctx* ctx, const std::exception& e) {
  if (ctx) ctx->err = e.what();
  g_err = e.what();
  return PSC_ERR_ARG;
}

#define API_BEGIN try {
#define API_END(ctx)                              \
  }                                               \
  catch (const Error& e) { return fail((ctx), e); } \
  catch (const std::bad_alloc&) { return fail((ctx), Error(PSC_ERR_NOMEM, "host allocation failed")); } \
  catch (const std::exception& e) { return fail((ctx), e); }

// make the library stream wait for everything already queued on the user stream
void enter(psc_ctx* ctx) {
  PSC_CUDA(cudaSetDevice(ctx->device));
  PSC_CUDA(cudaEventRecord(ctx->ev_user, ctx->user_stream));
  PSC_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_user, 0));
}

int64_t owner_of(const std::vector<int64_t>& rs, int64_t g) {
  return (int64_t)(std::upper_bound(rs.begin(), rs.end(), g) - rs.begin()) - 1;
}

}  // namespace

namespace psc {

// sorted unique off-rank halo + per-owner counts (host arithmetic of psb_cdasb)
void halo_plan(const std::vector<int64_t>& row_start, int rank, std::vector<int64_t>& refs,
               std::vector<int64_t>& rcount) {
  const int R = (int)row_start.size() - 1;
  const int64_t ob = row_start[rank], oe = row_start[rank + 1];
  refs.erase(std::remove_if(refs.begin(), refs.end(), [&](int64_t g) { return g >= ob && g < oe; }), refs.end());
  std::sort(refs.begin(), refs.end());
  refs.erase(std::unique(refs.begin(), refs.end()), refs.end());
  rcount.assign(R, 0);
  for (int64_t g : refs) {
    PSC_REQUIRE(g >= 0 && g < row_start[R], PSC_ERR_ARG, "halo column out of range");
    rcount[owner_of(row_start, g)]++;
  }
}

// requests of the peers (global, grouped by peer) -> local owned indices
void send_plan(const std::vector<int64_t>& row_start, int rank, const int64_t* req, int64_t n, int32_t* idx) {
  const int64_t ob = row_start[rank], no = row_start[rank + 1] - ob;
  for (int64_t k = 0; k < n; ++k) {
    const int64_t li = req[k] - ob;
    PSC_REQUIRE(li >= 0 && li < no, PSC_ERR_STATE, "halo request for a non-owned index");
    idx[k] = (int32_t)li;
  }
}

void desc_assemble(psc_desc* d) {
  psc_ctx* ctx = d->ctx;
  const int R = ctx->nranks;
  halo_plan(d->row_start, ctx->rank, d->halo_req, d->rcount);
  d->halo.swap(d->halo_req);
  std::vector<int64_t>().swap(d->halo_req);
  PSC_REQUIRE(d->n_own + d->n_halo() < (int64_t)INT32_MAX, PSC_ERR_ARG, "local index space exceeds int32");
  d->roff.assign(R + 1, 0);
  for (int p = 0; p < R; ++p) d->roff[p + 1] = d->roff[p] + d->rcount[p];
  d->scount.assign(R, 0);
  d->soff.assign(R + 1, 0);
  d->d_halo = dalloc<int64_t>(d->halo.size());
  if (!d->halo.empty())
    PSC_CUDA(cudaMemcpy(d->d_halo, d->halo.data(), sizeof(int64_t) * d->halo.size(), cudaMemcpyHostToDevice));
  if (R > 1) {
    cudaStream_t s = ctx->stream;
    // 1) every rank learns how many of its owned entries each peer needs
    int64_t* d_cnt = dalloc<int64_t>((size_t)R * (R + 1));
    PSC_CUDA(cudaMemcpyAsync(d_cnt + (size_t)R * R + 0, d->rcount.data(), sizeof(int64_t) * R,
                             cudaMemcpyHostToDevice, s));
    PSC_NCCL(ncclAllGather(d_cnt + (size_t)R * R, d_cnt, R, ncclInt64, ctx->comm, s));
    std::vector<int64_t> all((size_t)R * R);
    PSC_CUDA(cudaMemcpyAsync(all.data(), d_cnt, sizeof(int64_t) * R * R, cudaMemcpyDeviceToHost, s));
    PSC_CUDA(cudaStreamSynchronize(s));
    dfree(d_cnt);
    for (int p = 0; p < R; ++p) d->scount[p] = all[(size_t)p * R + ctx->rank];
    for (int p = 0; p < R; ++p) d->soff[p + 1] = d->soff[p] + d->scount[p];
    d->n_send = d->soff[R];
    PSC_REQUIRE(d->scount[ctx->rank] == 0 && d->rcount[ctx->rank] == 0, PSC_ERR_STATE, "self halo");
    // 2) requests (global indices) go to the owners
    int64_t* d_req = dalloc<int64_t>(d->n_send);
    PSC_NCCL(ncclGroupStart());
    for (int p = 0; p < R; ++p) {
      if (d->rcount[p]) PSC_NCCL(ncclSend(d->d_halo + d->roff[p], d->rcount[p], ncclInt64, p, ctx->comm, s));
      if (d->scount[p]) PSC_NCCL(ncclRecv(d_req + d->soff[p], d->scount[p], ncclInt64, p, ctx->comm, s));
    }
    PSC_NCCL(ncclGroupEnd());
    std::vector<int64_t> req(d->n_send);
    if (d->n_send)
      PSC_CUDA(cudaMemcpyAsync(req.data(), d_req, sizeof(int64_t) * d->n_send, cudaMemcpyDeviceToHost, s));
    PSC_CUDA(cudaStreamSynchronize(s));
    dfree(d_req);
    std::vector<int32_t> idx(d->n_send);
    send_plan(d->row_start, ctx->rank, req.data(), d->n_send, idx.data());
    d->d_send_idx = dalloc<int32_t>(idx.size());
    d->d_sendbuf = dalloc<double>(idx.size());
    if (!idx.empty())
      PSC_CUDA(cudaMemcpy(d->d_send_idx, idx.data(), sizeof(int32_t) * idx.size(), cudaMemcpyHostToDevice));
  } else {
    PSC_REQUIRE(d->halo.empty(), PSC_ERR_STATE, "halo on a single rank");
  }
  d->assembled = true;
}

// Halo exchange of an owned+halo vector of index space d (C1 in SURVEY.md):
// gather the entries the peers need (pack kernel) and receive the halo directly
// into its contiguous slots [n_own + roff[p], ...) — no unpack step.
void halo_exchange(psc_ctx* ctx, psc_desc* d, double* x, cudaStream_t s) {
  if (ctx->nranks == 1) return;
  if (d->n_send == 0 && d->halo.empty()) return;
  launch_pack(ctx, d->n_send, d->d_send_idx, x, d->d_sendbuf, s);
  PSC_NCCL(ncclGroupStart());
  for (int p = 0; p < ctx->nranks; ++p) {
    if (d->scount[p]) PSC_NCCL(ncclSend(d->d_sendbuf + d->soff[p], d->scount[p], ncclDouble, p, ctx->comm, s));
    if (d->rcount[p]) PSC_NCCL(ncclRecv(x + d->n_own + d->roff[p], d->rcount[p], ncclDouble, p, ctx->comm, s));
  }
  PSC_NCCL(ncclGroupEnd());
  ctx->collectives++;
}

void mat_assemble(psc_mat* m) {
  PSC_REQUIRE(m->rows->assembled && m->cols->assembled, PSC_ERR_STATE, "descriptors not assembled");
  PSC_REQUIRE(!m->assembled, PSC_ERR_STATE, "matrix already assembled");
  psc_desc* c = m->cols;
  sell_from_csr(m->ctx, m->n_rows, m->d_rowptr, m->d_colg, m->d_valcsr, m->nnz, c->own_begin, c->n_own, c->d_halo,
                c->n_halo(), m->S, m->ctx->stream, 0, m->rows == m->cols);
  dfree(m->d_rowptr);
  dfree(m->d_colg);
  dfree(m->d_valcsr);
  m->d_rowptr = nullptr;
  m->d_colg = nullptr;
  m->d_valcsr = nullptr;
  m->assembled = true;
}

}  // namespace psc

extern "C" {

const char* psc_version(void) {
  static std::string v = std::string("libpsc sm_100a nvcc ") + std::to_string(__CUDACC_VER_MAJOR__) + "." +
                         std::to_string(__CUDACC_VER_MINOR__) + " nccl-header " + std::to_string(NCCL_MAJOR) + "." +
                         std::to_string(NCCL_MINOR) + "." + std::to_string(NCCL_PATCH);
  return v.c_str();
}

const char* psc_status_string(int st) {
  switch (st) {
    case PSC_OK: return "PSC_OK";
    case PSC_NOT_CONVERGED: return "PSC_NOT_CONVERGED";
    case PSC_ERR_ARG: return "PSC_ERR_ARG";
    case PSC_ERR_STATE: return "PSC_ERR_STATE";
    case PSC_ERR_CUDA: return "PSC_ERR_CUDA";
    case PSC_ERR_NCCL: return "PSC_ERR_NCCL";
    case PSC_ERR_NOMEM: return "PSC_ERR_NOMEM";
    case PSC_ERR_BREAKDOWN: return "PSC_ERR_BREAKDOWN";
  }
  return "PSC_UNKNOWN_STATUS";
}

void* psc_ctx_stream(psc_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

const char* psc_last_error(psc_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

int psc_get_unique_id(unsigned char id[128]) {
  API_BEGIN
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  PSC_REQUIRE(id, PSC_ERR_ARG, "null id");
  ncclUniqueId u;
  PSC_NCCL(ncclGetUniqueId(&u));
  std::memcpy(id, &u, 128);
  return PSC_OK;
  API_END(nullptr)
}

int psc_init(int rank, int nranks, int cuda_device, const unsigned char* id, void* user_stream, psc_ctx** out) {
  psc_ctx* ctx = nullptr;
  API_BEGIN
  PSC_REQUIRE(out && nranks >= 1 && rank >= 0 && rank < nranks, PSC_ERR_ARG, "bad rank/nranks");
  PSC_REQUIRE(nranks == 1 || id, PSC_ERR_ARG, "nccl unique id required for nranks > 1");
  *out = nullptr;
  int ndev = 0;
  PSC_CUDA(cudaGetDeviceCount(&ndev));
  PSC_REQUIRE(cuda_device >= 0 && cuda_device < ndev, PSC_ERR_ARG, "bad cuda_device");
  PSC_CUDA(cudaSetDevice(cuda_device));
  cudaDeviceProp prop;
  PSC_CUDA(cudaGetDeviceProperties(&prop, cuda_device));
  PSC_REQUIRE(prop.major == 10 && prop.minor == 0, PSC_ERR_CUDA,
              std::string("libpsc is built for sm_100a (B200); device is ") + prop.name);
  ctx = new psc_ctx();
  ctx->rank = rank;
  ctx->nranks = nranks;
  ctx->device = cuda_device;
  ctx->num_sms = prop.multiProcessorCount;
  ctx->user_stream = static_cast<cudaStream_t>(user_stream);
  PSC_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  PSC_CUDA(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
  PSC_CUDA(cudaEventCreateWithFlags(&ctx->ev_user, cudaEventDisableTiming));
  if (nranks > 1) {
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    PSC_NCCL(ncclCommInitRank(&ctx->comm, nranks, u, rank));
  }
  *out = ctx;
  return PSC_OK;
  }
  catch (const Error& e) {
    if (ctx) psc_finalize(ctx);
    return fail(nullptr, e);
  }
  catch (const std::exception& e) {
    if (ctx) psc_finalize(ctx);
    return fail(nullptr, e);
  }
}

void psc_finalize(psc_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  if (ctx->ev_user) cudaEventDestroy(ctx->ev_user);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
  delete ctx;
}

int psc_halo_plan(int nranks, int rank, const int64_t* row_start, int64_t n_refs, const int64_t* refs, int64_t* halo,
                  int64_t* n_halo, int64_t* recv_count) {
  API_BEGIN
  PSC_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks && row_start && (refs || n_refs == 0) && n_halo &&
                  recv_count && (halo || n_refs == 0),
              PSC_ERR_ARG, "bad argument");
  std::vector<int64_t> rs(row_start, row_start + nranks + 1);
  PSC_REQUIRE(rs[0] == 0, PSC_ERR_ARG, "row_start[0] != 0");
  for (int r = 0; r < nranks; ++r) PSC_REQUIRE(rs[r] <= rs[r + 1], PSC_ERR_ARG, "row_start decreasing");
  std::vector<int64_t> v(refs, refs + n_refs);
  std::vector<int64_t> rc;
  halo_plan(rs, rank, v, rc);
  std::copy(v.begin(), v.end(), halo);
  *n_halo = (int64_t)v.size();
  std::copy(rc.begin(), rc.end(), recv_count);
  return PSC_OK;
  API_END(nullptr)
}

int psc_send_plan(int nranks, int rank, const int64_t* row_start, const int64_t* send_count, const int64_t* requests,
                  int32_t* send_idx) {
  API_BEGIN
  PSC_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks && row_start && send_count, PSC_ERR_ARG, "bad argument");
  std::vector<int64_t> rs(row_start, row_start + nranks + 1);
  int64_t n = 0;
  for (int p = 0; p < nranks; ++p) n += send_count[p];
  PSC_REQUIRE(n == 0 || (requests && send_idx), PSC_ERR_ARG, "null requests/send_idx");
  send_plan(rs, rank, requests, n, send_idx);
  return PSC_OK;
  API_END(nullptr)
}

int psc_desc_create(psc_ctx* ctx, int64_t n_global, const int64_t* row_start, psc_desc** out) {
  API_BEGIN
  PSC_REQUIRE(ctx && out && row_start && n_global >= 0, PSC_ERR_ARG, "bad argument");
  const int R = ctx->nranks;
  PSC_REQUIRE(row_start[0] == 0 && row_start[R] == n_global, PSC_ERR_ARG,
              "row_start must start at 0 and end at n_global");
  for (int r = 0; r < R; ++r) PSC_REQUIRE(row_start[r] <= row_start[r + 1], PSC_ERR_ARG, "row_start decreasing");
  psc_desc* d = new psc_desc();
  d->ctx = ctx;
  d->n_global = n_global;
  d->row_start.assign(row_start, row_start + R + 1);
  d->own_begin = row_start[ctx->rank];
  d->n_own = row_start[ctx->rank + 1] - row_start[ctx->rank];
  *out = d;
  return PSC_OK;
  API_END(ctx)
}

int psc_desc_assemble(psc_desc* d) {
  psc_ctx* ctx = d ? d->ctx : nullptr;
  API_BEGIN
  PSC_REQUIRE(d, PSC_ERR_ARG, "null descriptor");
  PSC_REQUIRE(!d->assembled, PSC_ERR_STATE, "descriptor already assembled");
  PSC_CUDA(cudaSetDevice(ctx->device));
  desc_assemble(d);
  return PSC_OK;
  API_END(ctx)
}

int psc_desc_info(psc_desc* d, int64_t* n_owned, int64_t* n_halo, int64_t* own_begin) {
  psc_ctx* ctx = d ? d->ctx : nullptr;
  API_BEGIN
  PSC_REQUIRE(d, PSC_ERR_ARG, "null descriptor");
  PSC_REQUIRE(d->assembled, PSC_ERR_STATE, "descriptor not assembled");
  if (n_owned) *n_owned = d->n_own;
  if (n_halo) *n_halo = d->n_halo();
  if (own_begin) *own_begin = d->own_begin;
  return PSC_OK;
  API_END(ctx)
}

int psc_desc_halo(psc_desc* d, int64_t* halo_globals) {
  psc_ctx* ctx = d ? d->ctx : nullptr;
  API_BEGIN
  PSC_REQUIRE(d && halo_globals, PSC_ERR_ARG, "null argument");
  PSC_REQUIRE(d->assembled, PSC_ERR_STATE, "descriptor not assembled");
  std::copy(d->halo.begin(), d->halo.end(), halo_globals);
  return PSC_OK;
  API_END(ctx)
}

void psc_desc_destroy(psc_desc* d) {
  if (!d) return;
  cudaSetDevice(d->ctx->device);
  dfree(d->d_send_idx);
  dfree(d->d_sendbuf);
  dfree(d->d_halo);
  delete d;
}

int psc_mat_create_csr(psc_ctx* ctx, psc_desc* rows, psc_desc* cols, int64_t n_local_rows, const int64_t* row_ptr,
                       const int64_t* col_global, const double* val, psc_mat** out) {
  psc_mat* m = nullptr;
  API_BEGIN
  PSC_REQUIRE(ctx && rows && cols && out && row_ptr, PSC_ERR_ARG, "null argument");
  PSC_REQUIRE(rows->ctx == ctx && cols->ctx == ctx, PSC_ERR_ARG, "descriptor of another context");
  PSC_REQUIRE(!cols->assembled, PSC_ERR_STATE, "column descriptor already assembled (create matrices first)");
  PSC_REQUIRE(n_local_rows == rows->n_own, PSC_ERR_ARG, "n_local_rows != owned rows of the row descriptor");
  PSC_REQUIRE(row_ptr[0] == 0, PSC_ERR_ARG, "row_ptr[0] != 0");
  for (int64_t i = 0; i < n_local_rows; ++i)
    PSC_REQUIRE(row_ptr[i + 1] >= row_ptr[i], PSC_ERR_ARG, "row_ptr decreasing");
  const int64_t nnz = row_ptr[n_local_rows];
  PSC_REQUIRE(nnz == 0 || (col_global && val), PSC_ERR_ARG, "null col/val");
  PSC_CUDA(cudaSetDevice(ctx->device));
  // validate + register off-rank columns as halo of `cols` (psb_spins)
  const int64_t ob = cols->own_begin, oe = cols->own_begin + cols->n_own, ng = cols->n_global;
  std::vector<int64_t> off;
  for (int64_t i = 0; i < n_local_rows; ++i) {
    int64_t prev = -1;
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      const int64_t g = col_global[k];
      PSC_REQUIRE(g > prev && g < ng, PSC_ERR_ARG,
                  "columns must be strictly increasing within a row and < n_global (row " + std::to_string(i) + ")");
      prev = g;
      if (g < ob || g >= oe) off.push_back(g);
    }
  }
  std::sort(off.begin(), off.end());
  off.erase(std::unique(off.begin(), off.end()), off.end());
  cols->halo_req.insert(cols->halo_req.end(), off.begin(), off.end());
  m = new psc_mat();
  m->ctx = ctx;
  m->rows = rows;
  m->cols = cols;
  m->n_rows = n_local_rows;
  m->nnz = nnz;
  m->d_rowptr = dalloc<int64_t>(n_local_rows + 1);
  m->d_colg = dalloc<int64_t>(nnz);
  m->d_valcsr = dalloc<double>(nnz);
  PSC_CUDA(cudaMemcpy(m->d_rowptr, row_ptr, sizeof(int64_t) * (n_local_rows + 1), cudaMemcpyHostToDevice));
  if (nnz) {
    PSC_CUDA(cudaMemcpy(m->d_colg, col_global, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice));
    PSC_CUDA(cudaMemcpy(m->d_valcsr, val, sizeof(double) * nnz, cudaMemcpyHostToDevice));
  }
  // small matrices keep a host copy (replicated coarse levels)
  if (nnz <= (int64_t)1 << 27) {
    m->h_rowptr.assign(row_ptr, row_ptr + n_local_rows + 1);
    m->h_colg.assign(col_global, col_global + nnz);
    m->h_val.assign(val, val + nnz);
  }
  *out = m;
  return PSC_OK;
  }
  catch (const Error& e) {
    psc_mat_destroy(m);
    return fail(ctx, e);
  }
  catch (const std::exception& e) {
    psc_mat_destroy(m);
    return fail(ctx, e);
  }
}

int psc_mat_assemble(psc_mat* m) {
  psc_ctx* ctx = m ? m->ctx : nullptr;
  API_BEGIN
  PSC_REQUIRE(m, PSC_ERR_ARG, "null matrix");
  PSC_CUDA(cudaSetDevice(ctx->device));
  mat_assemble(m);
  return PSC_OK;
  API_END(ctx)
}

int psc_mat_info(psc_mat* m, int64_t* nnz, int64_t* padded, int64_t* n_units, int64_t* n_rows, int* lanes) {
  psc_ctx* ctx = m ? m->ctx : nullptr;
  API_BEGIN
  PSC_REQUIRE(m, PSC_ERR_ARG, "null matrix");
  PSC_REQUIRE(m->assembled, PSC_ERR_STATE, "matrix not assembled");
  if (nnz) *nnz = m->nnz;
  if (padded) *padded = m->S.padded;
  if (n_units) *n_units = m->S.n_units;
  if (n_rows) *n_rows = m->n_rows;
  if (lanes) *lanes = m->S.lanes;
  return PSC_OK;
  API_END(ctx)
}

int psc_mat_spmv(psc_mat* m, double alpha, const double* x, double beta, double* y) {
  psc_ctx* ctx = m ? m->ctx : nullptr;
  API_BEGIN
  PSC_REQUIRE(m && (x || m->cols->n_own == 0) && (y || m->n_rows == 0), PSC_ERR_ARG, "null argument");
  PSC_REQUIRE(m->assembled, PSC_ERR_STATE, "matrix not assembled");
  enter(ctx);
  cudaStream_t s = ctx->stream;
  psc_desc* c = m->cols;
  double* xh = dalloc<double>(c->n_own + c->n_halo());
  if (c->n_own)
    PSC_CUDA(cudaMemcpyAsync(xh, x, sizeof(double) * c->n_own, cudaMemcpyDeviceToDevice, s));
  halo_exchange(ctx, c, xh, s);
  RowArgs a;
  a.alpha = alpha;
  a.beta = beta;
  a.x = xh;
  a.y = y;
  if (m->S.n_units) launch_rows(ctx, m->S, RowOp::Spmv, a, s);
  PSC_CUDA(cudaStreamSynchronize(s));
  dfree(xh);
  return PSC_OK;
  API_END(ctx)
}

int psc_mat_update_values(psc_mat* m, const double* val) {
  psc_ctx* ctx = m ? m->ctx : nullptr;
  double* d = nullptr;
  API_BEGIN
  PSC_REQUIRE(m && (val || m->nnz == 0), PSC_ERR_ARG, "null argument");
  PSC_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  if (!m->assembled) {
    if (m->nnz) PSC_CUDA(cudaMemcpyAsync(m->d_valcsr, val, sizeof(double) * m->nnz, cudaMemcpyHostToDevice, s));
  } else if (m->nnz) {
    d = dalloc<double>(m->nnz);
    PSC_CUDA(cudaMemcpyAsync(d, val, sizeof(double) * m->nnz, cudaMemcpyHostToDevice, s));
    sell_update_values(ctx, m->S, d, s);
  }
  if (!m->h_val.empty()) m->h_val.assign(val, val + m->nnz);
  PSC_CUDA(cudaStreamSynchronize(s));
  dfree(d);
  return PSC_OK;
  }
  catch (const Error& e) {
    dfree(d);
    return fail(ctx, e);
  }
  catch (const std::exception& e) {
    dfree(d);
    return fail(ctx, e);
  }
}

void psc_mat_destroy(psc_mat* m) {
  if (!m) return;
  cudaSetDevice(m->ctx->device);
  dfree(m->d_rowptr);
  dfree(m->d_colg);
  dfree(m->d_valcsr);
  sell_free(m->S);
  delete m;
}

}  // extern "C"
