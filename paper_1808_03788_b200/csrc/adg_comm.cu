// adg_comm.cu -- the multi-GPU exchange of the slab decomposition behind the
// C-ABI: an NCCL communicator bound to an adg_handle's
// device, the x-slab face-trace halo swap (grouped ncclSend / ncclRecv to the
// periodic ring neighbours) and the two reductions a step needs (the CFL
// record: MAX of the wave-speed bit patterns, SUM of the admissible /
// non-finite counts; conserved totals: SUM).  Everything is stream ordered on
// the caller's stream and CUDA-graph capturable; nothing synchronises the
// host.  The reference is single-process (driver.py:186-230); the exchange
// reproduces its periodic face states (driver.py:234-248) across the cut.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "adg_internal.h"

// NCCL is bound at run time, not at link time: the process's NCCL is the one
// torch.distributed already loaded (dlopen RTLD_NOLOAD finds it), else the
// system libnccl.so.2.  Linking it would let a process that loads this
// library before torch resolve torch's NCCL symbols against an older NCCL.
namespace {
struct NcclApi {
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommAbort) commAbort = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define ADG_NCCL_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
    ADG_NCCL_SYM(getUniqueId, "ncclGetUniqueId");
    ADG_NCCL_SYM(commInitRank, "ncclCommInitRank");
    ADG_NCCL_SYM(commAbort, "ncclCommAbort");
    ADG_NCCL_SYM(groupStart, "ncclGroupStart");
    ADG_NCCL_SYM(groupEnd, "ncclGroupEnd");
    ADG_NCCL_SYM(send, "ncclSend");
    ADG_NCCL_SYM(recv, "ncclRecv");
    ADG_NCCL_SYM(allReduce, "ncclAllReduce");
    ADG_NCCL_SYM(errorString, "ncclGetErrorString");
#undef ADG_NCCL_SYM
    api.ok = api.getUniqueId && api.commInitRank && api.commAbort && api.groupStart &&
             api.groupEnd && api.send && api.recv && api.allReduce && api.errorString;
  });
  return api;
}
}  // namespace

struct adg_comm {
  ncclComm_t nccl = nullptr;
  int nranks = 1;
  int rank = 0;
  int device = 0;
};

namespace adg {

static int nccl_fail(ncclResult_t r, std::string* err) {
  if (r == ncclSuccess) return ADG_OK;
  *err = std::string("NCCL: ") + nccl().errorString(r);
  return ADG_ERR_RUNTIME;
}

static bool nccl_missing(std::string* err) {
  if (nccl().ok) return false;
  *err = "NCCL (libnccl.so.2) is not available in this process";
  return true;
}

int comm_unique_id(void* out, std::string* err) {
  if (nccl_missing(err)) return ADG_ERR_RUNTIME;
  ncclUniqueId id;
  int rc = nccl_fail(nccl().getUniqueId(&id), err);
  if (rc == ADG_OK) std::memcpy(out, &id, sizeof(id));
  return rc;
}

int comm_init(int device, const void* uid, int nranks, int rank, adg_comm** out,
              std::string* err) {
  if (nccl_missing(err)) return ADG_ERR_RUNTIME;
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  adg_comm* c = new adg_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  int rc = nccl_fail(nccl().commInitRank(&c->nccl, nranks, id, rank), err);
  if (rc != ADG_OK) {
    delete c;
    return rc;
  }
  *out = c;
  return ADG_OK;
}

int comm_destroy(adg_comm* c) {
  if (!c) return ADG_OK;
  // every call on the communicator was stream ordered and the caller drops
  // it after its streams (and any CUDA graph holding its calls) are done:
  // abort frees the resources without the collective teardown handshake,
  // which can block when ranks (or interpreter shutdown) release out of step
  if (c->nccl) nccl().commAbort(c->nccl);
  delete c;
  return ADG_OK;
}

int comm_device(const adg_comm* c) { return c ? c->device : -1; }

// x-slab halo: this rank's low-x trace plane (first element layer) goes to
// rank-1 (its high ghost), the high-x plane (last layer) to rank+1 (its low
// ghost).  Traces are [d][2][E][tb]; a plane is the E / cells_x elements of
// one x-layer, contiguous in the C order of the grid.
int halo_exchange(adg_comm* c, const adg_grid* g, const double* traces, double* ghost_lo,
                  double* ghost_hi, cudaStream_t st, std::string* err) {
  int64_t pd = 1;
  for (int j = 0; j < g->dim; ++j) pd *= g->degree + 1;
  const int64_t blk = pd * g->nvars;
  const int64_t tb = blk + (blk & 1);
  const int64_t E = n_elements(g);
  const int64_t layer = E / g->cells[0];
  const size_t n = (size_t)(layer * tb);
  const double* lo_plane = traces;                              // axis 0, side 0, layer 0
  const double* hi_plane = traces + (size_t)(2 * E - layer) * tb;   // axis 0, side 1, last layer
  const int left = (c->rank - 1 + c->nranks) % c->nranks;
  const int right = (c->rank + 1) % c->nranks;
  ncclResult_t r = nccl().groupStart();
  if (r == ncclSuccess) r = nccl().send(lo_plane, n, ncclDouble, left, c->nccl, st);
  if (r == ncclSuccess) r = nccl().recv(ghost_hi, n, ncclDouble, right, c->nccl, st);
  if (r == ncclSuccess) r = nccl().send(hi_plane, n, ncclDouble, right, c->nccl, st);
  if (r == ncclSuccess) r = nccl().recv(ghost_lo, n, ncclDouble, left, c->nccl, st);
  ncclResult_t r2 = nccl().groupEnd();
  return nccl_fail(r != ncclSuccess ? r : r2, err);
}

// adg_reduce: lam_bits[3] MAX (bit patterns of non-negative doubles order
// like unsigned integers), n_admissible / n_nonfinite SUM
int allreduce_record(adg_comm* c, adg_reduce* red, cudaStream_t st, std::string* err) {
  uint64_t* w = reinterpret_cast<uint64_t*>(red);
  ncclResult_t r = nccl().groupStart();
  if (r == ncclSuccess) r = nccl().allReduce(w, w, 3, ncclUint64, ncclMax, c->nccl, st);
  if (r == ncclSuccess) r = nccl().allReduce(w + 3, w + 3, 2, ncclUint64, ncclSum, c->nccl, st);
  ncclResult_t r2 = nccl().groupEnd();
  return nccl_fail(r != ncclSuccess ? r : r2, err);
}

int allreduce_sum(adg_comm* c, double* buf, int64_t n, cudaStream_t st, std::string* err) {
  return nccl_fail(nccl().allReduce(buf, buf, (size_t)n, ncclDouble, ncclSum, c->nccl, st), err);
}

}  // namespace adg
