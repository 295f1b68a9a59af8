// a10/a11 — distributed runtime over NCCL (the MPI backend analogue).
//   halo exchange (exchange_ghost): pack owned boundary rows per peer (K-b7), then one
//     grouped ncclSend/ncclRecv per peer that lands straight in the ghost rows of the layer
//     buffer (local-then-ghost layout), so the paper's unpack step disappears.
//   gradient all-reduce: ncclAllReduce(sum) of the flat gradient buffer.
#include <nccl.h>

#include <cstring>

#include "internal.cuh"

struct mph_comm {
  ncclComm_t nccl = nullptr;
  int32_t world = 1, rank = 0;
};

namespace mph {
static int nccl_fail(ncclResult_t r, const char* what) {
  return fail(MPH_ENCCL, "%s: %s", what, ncclGetErrorString(r));
}
}  // namespace mph

using namespace mph;

extern "C" int mph_comm_unique_id(uint8_t* id_h) {
  if (!id_h) return fail(MPH_EINVAL, "null id");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id_h, &id, sizeof(id));
  return MPH_OK;
}

extern "C" int mph_comm_create(const uint8_t* id_h, int32_t world, int32_t rank, mph_comm** out) {
  if (!id_h || !out || world < 1 || rank < 0 || rank >= world) return fail(MPH_EINVAL, "comm_create arguments");
  *out = nullptr;
  ncclUniqueId id;
  std::memcpy(&id, id_h, sizeof(id));
  mph_comm* c = new mph_comm();
  c->world = world;
  c->rank = rank;
  ncclResult_t r = ncclCommInitRank(&c->nccl, world, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(r, "ncclCommInitRank");
  }
  *out = c;
  return MPH_OK;
}

extern "C" int mph_comm_info(const mph_comm* c, int32_t* world_h, int32_t* rank_h) {
  if (!c) return fail(MPH_EINVAL, "null comm");
  if (world_h) *world_h = c->world;
  if (rank_h) *rank_h = c->rank;
  return MPH_OK;
}

extern "C" int mph_comm_destroy(mph_comm* c) {
  if (!c) return MPH_OK;
  if (c->nccl) ncclCommDestroy(c->nccl);
  delete c;
  return MPH_OK;
}

namespace mph {

int halo_reserve(const mph_graph* gc, int w) {
  mph_graph* g = const_cast<mph_graph*>(gc);
  const size_t need = (size_t)g->n_send * w;
  if (need <= g->send_cap) return MPH_OK;
  dev_free(g->send_buf);
  g->send_buf = nullptr;
  g->send_cap = 0;
  MPH_TRY(dev_alloc(&g->send_buf, need));
  g->send_cap = need;
  return MPH_OK;
}

// K-b7: gather the owned boundary rows of every peer's send list into the send buffer.
int halo_pack(const mph_graph* g, const float* buf, int w, int ld, cudaStream_t s) {
  MPH_TRY(halo_reserve(g, w));
  return pack_rows(g->send_ids, g->n_send, buf, ld, w, g->send_buf, s);
}

// One grouped ncclSend/ncclRecv per peer; receives land in the ghost rows [n_rows, n_cols).
int halo_sendrecv(const mph_graph* g, mph_comm* c, float* buf, int w, int ld, cudaStream_t s) {
  ncclResult_t r = ncclGroupStart();
  for (int q = 0; q < g->world && r == ncclSuccess; ++q) {
    if (q == g->rank) continue;
    const int64_t ns = g->send_offset[q + 1] - g->send_offset[q];
    if (ns > 0) r = ncclSend(g->send_buf + g->send_offset[q] * w, (size_t)ns * w, ncclFloat, q, c->nccl, s);
    if (r == ncclSuccess && g->n_recv[q] > 0)
      r = ncclRecv(buf + ((int64_t)g->n_rows + g->recv_offset[q]) * ld, (size_t)g->n_recv[q] * w, ncclFloat, q,
                   c->nccl, s);
  }
  ncclResult_t r2 = ncclGroupEnd();
  if (r != ncclSuccess) return nccl_fail(r, "halo send/recv");
  if (r2 != ncclSuccess) return nccl_fail(r2, "ncclGroupEnd");
  return MPH_OK;
}

}  // namespace mph

extern "C" int mph_halo_exchange(const mph_graph* gc, mph_comm* c, float* buf_d, int32_t w, int32_t ld, void* stream) {
  if (!gc || !c || !buf_d) return fail(MPH_EINVAL, "halo_exchange: null argument");
  if (!gc->local) return fail(MPH_EINVAL, "halo_exchange: graph is not localized");
  if (gc->world != c->world || gc->rank != c->rank) return fail(MPH_EINVAL, "halo_exchange: graph/comm rank mismatch");
  if (w <= 0 || w % 4 || ld != w) return fail(MPH_EINVAL, "halo_exchange: needs ld == w, w % 4 == 0");
  cudaStream_t s = (cudaStream_t)stream;
  MPH_TRY(halo_pack(gc, buf_d, w, ld, s));
  return halo_sendrecv(gc, c, buf_d, w, ld, s);
}

extern "C" int mph_allreduce_sum(mph_comm* c, void* buf_d, int64_t n, int32_t is_double, void* stream) {
  if (!c || (!buf_d && n > 0) || n < 0) return fail(MPH_EINVAL, "allreduce: bad arguments");
  if (n == 0 || c->world == 1) return MPH_OK;
  ncclResult_t r = ncclAllReduce(buf_d, buf_d, (size_t)n, is_double ? ncclDouble : ncclFloat, ncclSum, c->nccl,
                                 (cudaStream_t)stream);
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
  return MPH_OK;
}
