// dist.cu -- the multi-GPU layer (include/flashrnn_dist.h).
//
// Shards are (head range x batch range) blocks from frnn_partition: rank =
// hp * bs + bp with hs head partitions and bs batch partitions.  The only
// collectives the path has run after the whole T loop:
//   * dR / dbias: sum over the bs ranks of one head partition (the sums over b
//     of engine.hpp:317, :327-330).  Each rank's gradient is widened to fp32,
//     ncclAllReduce'd in fp32 on the head partition's communicator
//     (ncclCommSplit by hp when both axes are sharded) and rounded once back
//     to the element type -- the cross-rank sum adds no rounding of its own.
//   * activations / gradients: ncclAllGather of each rank's shard (padded to
//     the largest shard: ragged batch splits) into a [world][shard] staging
//     area, then one placement kernel writes every block into the full tensor
//     at its (batch, column) offsets.
// NCCL is dlopen'ed (libnccl.so.2) so single-GPU users never load it and a
// process that already has NCCL (PyTorch) shares that one library.
#include <cuda_bf16.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/flashrnn_debug.h"
#include "../../include/flashrnn_dist.h"
#include "kernels.h"

namespace {

using frnn::align_up;
using frnn::set_error;

struct Nccl {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* path = std::getenv("FRNN_NCCL_LIB");
    void* h = dlopen(path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.why = std::string("cannot load NCCL: ") + dlerror();
      return;
    }
    auto sym = [&](auto& fp, const char* name) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
      return fp != nullptr;
    };
    bool ok = sym(n.GetUniqueId, "ncclGetUniqueId") && sym(n.CommInitRank, "ncclCommInitRank") &&
              sym(n.CommDestroy, "ncclCommDestroy") && sym(n.AllReduce, "ncclAllReduce") &&
              sym(n.AllGather, "ncclAllGather") && sym(n.GroupStart, "ncclGroupStart") &&
              sym(n.GroupEnd, "ncclGroupEnd") && sym(n.GetErrorString, "ncclGetErrorString") &&
              sym(n.GetVersion, "ncclGetVersion");
    sym(n.CommSplit, "ncclCommSplit");  // optional (NCCL >= 2.18): mixed head x batch sharding
    n.ok = ok;
    if (!ok) n.why = "NCCL library lacks a required symbol";
  });
  return n;
}

int nccl_fail(ncclResult_t r, const char* what) {
  return set_error(FRNN_ECUDA, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace

struct frnn_dist {
  ncclComm_t comm = nullptr;   // all ranks
  ncclComm_t group = nullptr;  // ranks of this head partition (== comm when heads are not sharded)
  int world = 1, rank = 0, device = 0;
  bool owns = false;
  int group_hs = -1;           // head-partition count `group` was split for
};

namespace {

__global__ void widen_kernel(const __nv_bfloat16* in, float* out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = __bfloat162float(in[i]);
}
__global__ void narrow_kernel(const float* in, __nv_bfloat16* out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16_rn(in[i]);
}

// dst[((r*B + b0 + b)*J + j)*D + e0 + e] = src[((r*nb + b)*J + j)*ne + e]
// (element size 2 or 4 bytes; one thread per element, rows of the block in order)
template <class E>
__global__ void place_kernel(const E* src, E* dst, long long R, int nb, int J, int ne, int B, int D, int b0, int e0) {
  const long long n = R * nb * J * ne;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(i % ne);
    long long q = i / ne;
    const int j = (int)(q % J);
    q /= J;
    const int b = (int)(q % nb);
    const long long r = q / nb;
    dst[((r * B + b0 + b) * J + j) * D + e0 + e] = src[i];
  }
}

int grid_for(long long n) { return (int)std::min<long long>(148 * 8, (n + 255) / 256); }

cudaError_t place(const void* src, void* dst, size_t esz, long long R, int nb, int J, int ne, int B, int D, int b0,
                  int e0, cudaStream_t s) {
  const long long n = R * nb * J * ne;
  if (n == 0) return cudaSuccess;
  if (esz == 2)
    place_kernel<uint16_t><<<grid_for(n), 256, 0, s>>>(static_cast<const uint16_t*>(src), static_cast<uint16_t*>(dst),
                                                       R, nb, J, ne, B, D, b0, e0);
  else
    place_kernel<uint32_t><<<grid_for(n), 256, 0, s>>>(static_cast<const uint32_t*>(src), static_cast<uint32_t*>(dst),
                                                       R, nb, J, ne, B, D, b0, e0);
  return cudaGetLastError();
}

struct Layout {
  int hs, bs;  // head / batch partitions (frnn_partition's factorisation)
};
Layout layout_of(const frnn_dist* d, frnn_shape sh) {
  frnn_shard s0{};
  frnn_partition(sh, d->world, 0, &s0);
  const int hper = s0.head_end - s0.head_begin;
  const int hs = sh.num_heads / std::max(1, hper);
  return {hs, d->world / hs};
}

int check_common(const frnn_dist* d, const frnn_cell* cell, frnn_shape sh, int32_t dtype) {
  if (!d || !cell) return set_error(FRNN_EINVAL_ARG, "null argument");
  if (dtype != FRNN_F32 && dtype != FRNN_BF16) return set_error(FRNN_EUNSUPPORTED, "dtype must be f32 or bf16");
  frnn_shard s{};
  const int rc = frnn_partition(sh, d->world, d->rank, &s);
  if (rc) return rc;
  return FRNN_OK;
}

// The head-partition communicator (created on first use for a given split).
int head_group(frnn_dist* d, const Layout& L, ncclComm_t* out) {
  if (L.hs == 1) {
    *out = d->comm;
    return FRNN_OK;
  }
  if (d->group && d->group_hs == L.hs) {
    *out = d->group;
    return FRNN_OK;
  }
  if (!nccl().CommSplit) return set_error(FRNN_EUNSUPPORTED, "mixed head x batch sharding needs ncclCommSplit");
  if (d->group && d->group != d->comm) nccl().CommDestroy(d->group);
  d->group = nullptr;
  const int hp = d->rank / L.bs;
  ncclResult_t r = nccl().CommSplit(d->comm, hp, d->rank, &d->group, nullptr);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommSplit");
  d->group_hs = L.hs;
  *out = d->group;
  return FRNN_OK;
}

size_t shard_elems_max(const frnn_dist* d, frnn_shape sh, size_t per_row_col) {
  size_t mx = 0;
  for (int r = 0; r < d->world; ++r) {
    frnn_shard s{};
    frnn_partition(sh, d->world, r, &s);
    mx = std::max(mx, (size_t)(s.batch_end - s.batch_begin) * (s.head_end - s.head_begin) * per_row_col);
  }
  return mx;
}

// Elements of tensor k (0 states, 1 gates, 2 dx, 3 ds0, 4 dR, 5 dbias) in rank r's shard.
size_t shard_elems(const frnn_cell& c, frnn_shape sh, int world, int r, int k) {
  frnn_shard s{};
  frnn_partition(sh, world, r, &s);
  const size_t h = s.head_end - s.head_begin, b = s.batch_end - s.batch_begin, DH = sh.head_dim;
  const size_t NS = c.num_states, NG = c.num_gates, T = sh.seq_len;
  switch (k) {
    case 0: return (T + 1) * NS * b * h * DH;
    case 1: return T * NG * b * h * DH;
    case 2: return T * b * NG * h * DH;
    case 3: return NS * b * h * DH;
    case 4: return h * NG * DH * DH;
    default: return NG * h * DH;
  }
}

// Staging [world][blk] (every rank's shard of tensor k) -> the full tensor.
cudaError_t place_tensor(const frnn_cell& c, frnn_shape sh, int world, int k, size_t esz, const void* stage,
                         size_t blk, void* full, cudaStream_t st) {
  const int NS = c.num_states, NG = c.num_gates, T = sh.seq_len, B = sh.batch, DH = sh.head_dim;
  const int D = sh.num_heads * DH;
  for (int q = 0; q < world; ++q) {
    frnn_shard s{};
    frnn_partition(sh, world, q, &s);
    const int h0 = s.head_begin, h = s.head_end - s.head_begin, b0 = s.batch_begin, nb = s.batch_end - b0;
    const char* src = static_cast<const char*>(stage) + (size_t)q * blk * esz;
    cudaError_t e = cudaSuccess;
    switch (k) {
      case 0: e = place(src, full, esz, (long long)(T + 1) * NS, nb, 1, h * DH, B, D, b0, h0 * DH, st); break;
      case 1: e = place(src, full, esz, (long long)T * NG, nb, 1, h * DH, B, D, b0, h0 * DH, st); break;
      case 2: e = place(src, full, esz, T, nb, NG, h * DH, B, D, b0, h0 * DH, st); break;
      case 3: e = place(src, full, esz, NS, nb, 1, h * DH, B, D, b0, h0 * DH, st); break;
      case 4:  // [h][NG][DH][DH]: contiguous head slices; every batch shard holds the same (reduced) sum
        if (b0 == 0)
          e = cudaMemcpyAsync(static_cast<char*>(full) + (size_t)h0 * NG * DH * DH * esz, src,
                              (size_t)h * NG * DH * DH * esz, cudaMemcpyDeviceToDevice, st);
        break;
      default:  // [NG][e]: column slice of [NG][D]
        if (b0 == 0) e = place(src, full, esz, NG, 1, 1, h * DH, 1, D, 0, h0 * DH, st);
    }
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace

extern "C" {

int frnn_dist_nccl_version(void) {
  Nccl& n = nccl();
  int v = 0;
  if (!n.ok || n.GetVersion(&v) != ncclSuccess) return 0;
  return v;
}

int frnn_dist_unique_id(uint8_t id[128]) {
  frnn::clear_error();
  if (!id) return set_error(FRNN_EINVAL_ARG, "null id");
  Nccl& n = nccl();
  if (!n.ok) return set_error(FRNN_EUNSUPPORTED, n.why);
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId u;
  ncclResult_t r = n.GetUniqueId(&u);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id, &u, 128);
  return FRNN_OK;
}

int frnn_dist_init(const uint8_t id[128], int32_t world_size, int32_t rank, frnn_dist** out) {
  frnn::clear_error();
  if (!id || !out) return set_error(FRNN_EINVAL_ARG, "null argument");
  if (world_size < 1 || rank < 0 || rank >= world_size) return set_error(FRNN_EINVAL_ARG, "bad rank/world size");
  Nccl& n = nccl();
  if (!n.ok) return set_error(FRNN_EUNSUPPORTED, n.why);
  auto* d = new frnn_dist;
  d->world = world_size;
  d->rank = rank;
  d->owns = true;
  cudaGetDevice(&d->device);
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclResult_t r = n.CommInitRank(&d->comm, world_size, u, rank);
  if (r != ncclSuccess) {
    delete d;
    return nccl_fail(r, "ncclCommInitRank");
  }
  *out = d;
  return FRNN_OK;
}

int frnn_dist_from_comm(void* nccl_comm, int32_t world_size, int32_t rank, frnn_dist** out) {
  frnn::clear_error();
  if (!nccl_comm || !out) return set_error(FRNN_EINVAL_ARG, "null argument");
  if (world_size < 1 || rank < 0 || rank >= world_size) return set_error(FRNN_EINVAL_ARG, "bad rank/world size");
  if (!nccl().ok) return set_error(FRNN_EUNSUPPORTED, nccl().why);
  auto* d = new frnn_dist;
  d->comm = static_cast<ncclComm_t>(nccl_comm);
  d->world = world_size;
  d->rank = rank;
  cudaGetDevice(&d->device);
  *out = d;
  return FRNN_OK;
}

int frnn_dist_destroy(frnn_dist* d) {
  frnn::clear_error();
  if (!d) return FRNN_OK;
  if (d->group && d->group != d->comm) nccl().CommDestroy(d->group);
  if (d->owns && d->comm) nccl().CommDestroy(d->comm);
  delete d;
  return FRNN_OK;
}

int frnn_dist_shard(const frnn_dist* d, frnn_shape shape, frnn_shard* out) {
  frnn::clear_error();
  if (!d) return set_error(FRNN_EINVAL_ARG, "null argument");
  return frnn_partition(shape, d->world, d->rank, out);
}

int frnn_dist_workspace_size(const frnn_dist* d, const frnn_cell* cell, frnn_shape sh, int32_t dtype, size_t* bytes) {
  frnn::clear_error();
  if (!bytes) return set_error(FRNN_EINVAL_ARG, "null output");
  int rc = check_common(d, cell, sh, dtype);
  if (rc) return rc;
  const size_t esz = dtype == FRNN_BF16 ? 2 : 4;
  const size_t NS = cell->num_states, NG = cell->num_gates, T = sh.seq_len, DH = sh.head_dim;
  frnn_shard s{};
  frnn_partition(sh, d->world, d->rank, &s);
  const size_t h = s.head_end - s.head_begin;
  const size_t reduce = align_up(4 * (h * NG * DH * DH), 256) + align_up(4 * (NG * h * DH), 256);
  // gather staging: [world][largest shard] of the biggest tensor (states or gates, or dx), + one send block
  const size_t per = std::max({(T + 1) * NS, T * NG, NS}) * DH;  // elements per (batch row x head)
  const size_t blk = shard_elems_max(d, sh, per);
  const size_t pblk = std::max(NG * DH * DH, NG * DH) * (size_t)std::max(1, sh.num_heads);  // dR/db upper bound
  const size_t gather = align_up(esz * std::max(blk, pblk) * (d->world + 1), 256);
  *bytes = std::max(reduce, gather);
  return FRNN_OK;
}

int frnn_dist_reduce_param_grads(frnn_dist* d, const frnn_cell* cell, frnn_shape sh, int32_t dtype, void* dR,
                                 void* dbias, void* ws, size_t ws_bytes, void* stream) {
  frnn::clear_error();
  int rc = check_common(d, cell, sh, dtype);
  if (rc) return rc;
  if (!dR || !dbias) return set_error(FRNN_EINVAL_ARG, "null gradient pointer");
  const Layout L = layout_of(d, sh);
  // batch not sharded: nothing to sum (FRNN_DIST_FORCE_REDUCE=1 runs the collective anyway: a test hook)
  if (L.bs == 1 && !std::getenv("FRNN_DIST_FORCE_REDUCE")) return FRNN_OK;
  size_t need = 0;
  if ((rc = frnn_dist_workspace_size(d, cell, sh, dtype, &need))) return rc;
  if (dtype == FRNN_BF16 && (!ws || ws_bytes < need)) return set_error(FRNN_EINVAL_ARG, "workspace too small");
  ncclComm_t g = nullptr;
  if ((rc = head_group(d, L, &g))) return rc;
  frnn_shard s{};
  frnn_partition(sh, d->world, d->rank, &s);
  const size_t h = s.head_end - s.head_begin, NG = cell->num_gates, DH = sh.head_dim;
  const size_t nR = h * NG * DH * DH, nb = NG * h * DH;
  auto st = static_cast<cudaStream_t>(stream);
  Nccl& n = nccl();
  if (dtype == FRNN_F32) {
    ncclResult_t r = n.GroupStart();
    if (r == ncclSuccess) r = n.AllReduce(dR, dR, nR, ncclFloat32, ncclSum, g, st);
    if (r == ncclSuccess) r = n.AllReduce(dbias, dbias, nb, ncclFloat32, ncclSum, g, st);
    ncclResult_t r2 = n.GroupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess) return nccl_fail(r != ncclSuccess ? r : r2, "ncclAllReduce");
    return FRNN_OK;
  }
  float* wR = static_cast<float*>(ws);
  float* wb = reinterpret_cast<float*>(static_cast<char*>(ws) + align_up(4 * nR, 256));
  widen_kernel<<<grid_for(nR), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(dR), wR, nR);
  widen_kernel<<<grid_for(nb), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(dbias), wb, nb);
  ncclResult_t r = n.GroupStart();
  if (r == ncclSuccess) r = n.AllReduce(wR, wR, nR, ncclFloat32, ncclSum, g, st);
  if (r == ncclSuccess) r = n.AllReduce(wb, wb, nb, ncclFloat32, ncclSum, g, st);
  ncclResult_t r2 = n.GroupEnd();
  if (r != ncclSuccess || r2 != ncclSuccess) return nccl_fail(r != ncclSuccess ? r : r2, "ncclAllReduce");
  narrow_kernel<<<grid_for(nR), 256, 0, st>>>(wR, static_cast<__nv_bfloat16*>(dR), nR);
  narrow_kernel<<<grid_for(nb), 256, 0, st>>>(wb, static_cast<__nv_bfloat16*>(dbias), nb);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(FRNN_ECUDA, cudaGetErrorString(e));
  return FRNN_OK;
}

int frnn_dist_gather(frnn_dist* d, const frnn_cell* cell, frnn_shape sh, int32_t dtype, const frnn_dist_tensors* t,
                     void* ws, size_t ws_bytes, void* stream) {
  frnn::clear_error();
  int rc = check_common(d, cell, sh, dtype);
  if (rc) return rc;
  if (!t) return set_error(FRNN_EINVAL_ARG, "null tensors");
  size_t need = 0;
  if ((rc = frnn_dist_workspace_size(d, cell, sh, dtype, &need))) return rc;
  if (!ws || ws_bytes < need) return set_error(FRNN_EINVAL_ARG, "workspace too small");
  const size_t esz = dtype == FRNN_BF16 ? 2 : 4;
  auto st = static_cast<cudaStream_t>(stream);
  const void* loc[6] = {t->states, t->gates, t->dx, t->ds0, t->dR, t->dbias};
  void* full[6] = {t->states_full, t->gates_full, t->dx_full, t->ds0_full, t->dR_full, t->dbias_full};
  for (int k = 0; k < 6; ++k) {
    if (!loc[k] || !full[k]) continue;
    size_t blk = 0;
    for (int r = 0; r < d->world; ++r) blk = std::max(blk, shard_elems(*cell, sh, d->world, r, k));
    char* stage = static_cast<char*>(ws);
    char* send = stage + blk * esz * d->world;
    cudaError_t e = cudaMemcpyAsync(send, loc[k], shard_elems(*cell, sh, d->world, d->rank, k) * esz,
                                    cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return set_error(FRNN_ECUDA, cudaGetErrorString(e));
    ncclResult_t r = nccl().AllGather(send, stage, blk * esz, ncclUint8, d->comm, st);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
    e = place_tensor(*cell, sh, d->world, k, esz, stage, blk, full[k], st);
    if (e != cudaSuccess) return set_error(FRNN_ECUDA, cudaGetErrorString(e));
  }
  return FRNN_OK;
}

// Test hook: the placement half of frnn_dist_gather for a `world`-rank layout,
// from a staging buffer [world][blk] filled by the caller as ncclAllGather would
// (tensor k: 0 states, 1 gates, 2 dx, 3 ds0, 4 dR, 5 dbias); *blk_out = blk.
int frnn_debug_dist_place(const frnn_cell* cell, frnn_shape sh, int32_t dtype, int32_t world, int32_t k,
                          const void* stage, void* full, size_t* blk_out, void* stream) {
  frnn::clear_error();
  if (!cell || world < 1 || k < 0 || k > 5) return set_error(FRNN_EINVAL_ARG, "bad argument");
  size_t blk = 0;
  for (int r = 0; r < world; ++r) {
    frnn_shard s{};
    const int rc = frnn_partition(sh, world, r, &s);
    if (rc) return rc;
    blk = std::max(blk, shard_elems(*cell, sh, world, r, k));
  }
  if (blk_out) *blk_out = blk;
  if (!stage || !full) return FRNN_OK;
  const cudaError_t e = place_tensor(*cell, sh, world, k, dtype == FRNN_BF16 ? 2 : 4, stage, blk, full,
                                     static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return set_error(FRNN_ECUDA, cudaGetErrorString(e));
  return FRNN_OK;
}

}  // extern "C"
