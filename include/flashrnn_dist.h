/*
 * flashrnn_dist.h -- multi-GPU layer of libflashrnn.so, no PyTorch.
 *
 * The recurrence shards by batch x head with NO per-step communication
 * (heads never mix, engine.hpp:139-142; batch rows are independent except the
 * sums over b of dR and db, engine.hpp:317, :327-330).  Every rank runs
 * frnn_forward / frnn_backward on its shard (frnn_partition); this layer adds
 * the only collectives the path has, over NCCL (NVLink/NVSwitch on one box):
 *   - frnn_dist_reduce_param_grads: dR and dbias summed across the batch
 *     shards of the same head range (ncclAllReduce in fp32 of the per-rank
 *     bf16/fp32 gradients, rounded once back to the element type);
 *   - frnn_dist_gather: the sharded states / gates / dx / ds0 (and the head
 *     slices of dR / dbias) assembled into full-size tensors on every rank
 *     (ncclAllGather + one placement kernel per tensor).
 *
 * NCCL is loaded on first use (dlopen "libnccl.so.2"; FRNN_NCCL_LIB overrides).
 * In a process that already loaded NCCL (e.g. PyTorch's) that same library is
 * used, so a caller's own ncclComm_t can be wrapped with frnn_dist_from_comm.
 * All tensors are device pointers in rnnkit layouts (flashrnn.h); `shape` is
 * always the GLOBAL shape, local tensors are the rank's shard of it.
 * Reference interface this replaces: none -- rnnkit is single-process; the
 * partition/collective contract is SURVEY 8e (the reference's
 * engine.hpp:139-142, :317, :327-330 define what may be split).
 */
#ifndef FLASHRNN_DIST_H_
#define FLASHRNN_DIST_H_

#include "flashrnn.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct frnn_dist frnn_dist;  /* communicator(s) + rank/world + device */

/* ncclGetUniqueId: rank 0 creates the 128-byte id, the caller broadcasts it. */
FRNN_API int frnn_dist_unique_id(uint8_t id[128]);
/* ncclCommInitRank on the current CUDA device; the library owns the communicator. */
FRNN_API int frnn_dist_init(const uint8_t id[128], int32_t world_size, int32_t rank, frnn_dist** out);
/* Wrap the caller's ncclComm_t (must come from the same libnccl this process loaded). */
FRNN_API int frnn_dist_from_comm(void* nccl_comm, int32_t world_size, int32_t rank, frnn_dist** out);
FRNN_API int frnn_dist_destroy(frnn_dist* d);
/* NCCL version linked at run time (e.g. 22809), 0 if NCCL could not be loaded. */
FRNN_API int frnn_dist_nccl_version(void);

/* In place: dR [h_local][NG][DH][DH] and dbias [NG][h_local*DH] summed over the
 * ranks sharing this rank's head range (no-op when the batch is not sharded).
 * `workspace` >= frnn_dist_workspace_size bytes. */
FRNN_API int frnn_dist_reduce_param_grads(frnn_dist* d, const frnn_cell* cell, frnn_shape shape, int32_t dtype,
                                          void* dR, void* dbias, void* workspace, size_t workspace_bytes,
                                          void* stream);

/* Full-size outputs on every rank from the local shards.  Any pointer pair may
 * be NULL to skip that tensor.  Local (b = shard rows, e = shard columns):
 *   states [T+1][NS][b][e], gates [T][NG][b][e], dx [T][b][NG][e], ds0 [NS][b][e],
 *   dR [h][NG][DH][DH], dbias [NG][e]   (dR/dbias already reduced across batch shards)
 * Full: the same tensors at the global shape. */
typedef struct {
  const void *states, *gates, *dx, *ds0, *dR, *dbias;  /* local shard */
  void *states_full, *gates_full, *dx_full, *ds0_full, *dR_full, *dbias_full;
} frnn_dist_tensors;
FRNN_API int frnn_dist_gather(frnn_dist* d, const frnn_cell* cell, frnn_shape shape, int32_t dtype,
                              const frnn_dist_tensors* t, void* workspace, size_t workspace_bytes, void* stream);

/* Scratch for reduce (fp32 copy of dR + dbias) and gather (world x largest shard). */
FRNN_API int frnn_dist_workspace_size(const frnn_dist* d, const frnn_cell* cell, frnn_shape shape, int32_t dtype,
                                      size_t* bytes);
/* This rank's shard of `shape` (= frnn_partition(shape, world, rank)). */
FRNN_API int frnn_dist_shard(const frnn_dist* d, frnn_shape shape, frnn_shard* out);

#ifdef __cplusplus
}
#endif
#endif /* FLASHRNN_DIST_H_ */
