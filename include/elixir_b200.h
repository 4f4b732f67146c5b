/*
 * elixir_b200.h — C-ABI of the B200-native Elixir chunk-memory hot path.
 *
 * The reference (`/root/reference/pkg/src/offplan`, "offplan") is a pure-Python
 * planner/simulator. It specifies the runtime only through contracts:
 *   - layout:   pack_chunks            (offplan/chunking.py:102-138)
 *   - trace:    build_chunk_trace      (offplan/chunking.py:149-170)
 *   - schedule: simulate               (offplan/rcache_sim.py:87-199)
 *   - memory:   chunk_footprint        (offplan/cost_model.py:147-153)
 *   - update:   v_g / v_c velocities   (offplan/rcache_sim.py:173-184)
 * and through the paper's runtime prose (PAPER.md:170-181, :203-206, :221-238,
 * :276-281). Each entry point below names the reference interface it replaces
 * or implements. INTEGRATION.md shows the ctypes binding a maintainer adds.
 *
 * Conventions
 *   - Every buffer is caller-owned (torch tensors on the Python side). The
 *     library never allocates device memory.
 *   - Every GPU call is asynchronous on the `stream` argument (a cudaStream_t
 *     passed as void*). Cross-stream ordering is the caller's (events).
 *   - Return value: ELX_OK (0) or an elx_status error code; a thread-local
 *     message is available from elx_last_error(). No C++ exception crosses
 *     the ABI.
 *   - Element dtypes: ELX_F32, ELX_BF16, ELX_F16.
 *   - Not thread-safe per stream; one host thread per rank process.
 */
#ifndef ELIXIR_B200_H
#define ELIXIR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ELX_ABI_VERSION 1
#define ELX_MAX_WORLD 16

/* Status codes. The split mirrors offplan/errors.py:10-47:
 * ValidationError family -> 1xx, InfeasibleError family -> 2xx. */
typedef enum {
  ELX_OK = 0,
  ELX_ERR_VALIDATION = 100,        /* errors.py:14  ValidationError        */
  ELX_ERR_INFEASIBLE = 200,        /* errors.py:30  InfeasibleError        */
  ELX_ERR_CHUNK_TOO_SMALL = 201,   /* errors.py:34  ChunkTooSmallError     */
  ELX_ERR_INFEASIBLE_CACHE = 202,  /* errors.py:38  InfeasibleCacheError   */
  ELX_ERR_CUDA = 300,              /* CUDA runtime failure (no reference analogue) */
} elx_status;

typedef enum { ELX_F32 = 0, ELX_BF16 = 1, ELX_F16 = 2 } elx_dtype;

/* ---------------------------------------------------------------- misc */
int32_t elx_abi_version(void);
const char* elx_last_error(void);
/* Number of kernels this library launched in this process (all streams).
 * bench.py reports the delta over its timed region as `gpu_launches`. */
int64_t elx_launch_count(void);
/* Record a (timing) cudaEvent_t on a stream. Outside a capture this is
 * cudaEventRecord; while the stream is being captured into a CUDA graph the
 * record is EXTERNAL (an event-record node), so every replay of the graph
 * re-records the event and kernels inside a replayed step can be timed
 * (bench.py times K4 inside its timed graph replays this way). */
int elx_event_record(void* event, void* stream);
/* sizeof of the ABI structs, for binding checks: 0 elx_event, 1
 * elx_sim_counters, 2 elx_member, 3 elx_adam_seg, 4 elx_adam_hp,
 * 5 elx_cpu_seg; -1 for an unknown id. */
int64_t elx_sizeof(int32_t which);

/* ------------------------------------------------- host: layout + schedule
 *
 * elx_layout_pack replaces offplan.pack_chunks (chunking.py:102-138):
 * greedy in-order packing of `n` parameters (numel[i], already in the
 * packing order of partition_multiuse, chunking.py:82-99) into chunks of
 * `chunk_length` elements; a parameter never straddles two chunks.
 * Outputs: chunk_of[i], offset[i] (element offset inside the chunk), and
 * *n_chunks. Errors: chunk_length < 1 -> ELX_ERR_VALIDATION;
 * numel[i] > chunk_length -> ELX_ERR_CHUNK_TOO_SMALL (message names i). */
int elx_layout_pack(const int64_t* numel, int32_t n, int64_t chunk_length,
                    int32_t* chunk_of, int64_t* offset, int32_t* n_chunks);

/* One runtime event of the rCache program. Walk positions 0..F-1 are the
 * forward nodes, F..2F-1 the mirrored backward nodes (chunking.py:165). */
typedef enum { ELX_EV_GATHER = 0, ELX_EV_REDUCE = 1 } elx_event_kind;

typedef struct {
  int32_t kind;       /* elx_event_kind                                    */
  int32_t pos;        /* walk position at which the event is due           */
  int32_t chunk;      /* chunk id                                          */
  int32_t block;      /* rCache block the chunk occupies                   */
  int32_t victim;     /* chunk evicted from `block` (-1 = block was free)  */
  int32_t issue_pos;  /* earliest walk position the gather may be issued
                         at (prefetch); == pos if none   */
} elx_event;

/* Counter block with the field meaning of offplan.SimReport
 * (rcache_sim.py:65-84); byte fields are derived by the caller as
 * units * compute_bytes * chunk_length exactly as rcache_sim.py:186-199. */
typedef struct {
  int64_t gather_ops;
  int64_t replaced_ops;      /* gathers of a chunk already gathered once   */
  int64_t reduce_ops;
  int64_t c2g_units;         /* gathers of CPU-home chunks                 */
  int64_t g2c_units;         /* reduces of CPU-home chunks                 */
  int64_t peak_rcache_blocks;
  int64_t working_set;       /* chunking.py:173-177                        */
} elx_sim_counters;

/* elx_schedule replaces offplan.simulate's walk (rcache_sim.py:87-199) and
 * compiles it into an event program the runtime replays.
 *   forward nodes in CSR form: node i touches chunks
 *     node_chunks[node_ptr[i] .. node_ptr[i+1]) ;
 *   cpu_home[c] != 0 marks chunk c as CPU-homed (Device.CPU);
 *   events: capacity `events_cap`; *n_events receives the count (the call
 *     fails with ELX_ERR_VALIDATION if the capacity is too small).
 * Eviction: farthest next use, ties to the lowest chunk id; chunks are
 * pinned from their first backward touch until their reduce position.
 * Errors: ELX_ERR_VALIDATION (bad arguments), ELX_ERR_INFEASIBLE_CACHE
 * (n_block below the working set, or pinned chunks fill all blocks). */
int elx_schedule(int32_t n_nodes, const int32_t* node_ptr, const int32_t* node_chunks,
                 int32_t n_chunks, int32_t n_block, const uint8_t* cpu_home,
                 elx_event* events, int64_t events_cap, int64_t* n_events,
                 elx_sim_counters* counters);

/* ------------------------------------------------------- K1 chunk pack
 * Scatter parameters into a chunk buffer at their layout offsets (and the
 * reverse), the storage side of pack_chunks (chunking.py:113-131) and of
 * "we use the gradient to overwrite the data in the parameter chunk"
 * (PAPER.md:233-236). One call handles any number of members; `members` is
 * a HOST array (the library batches it into kernel parameters, so no device
 * table and no host->device copy is needed).
 *   ext:        external tensor pointer (param, grad, or export target);
 *               NULL in elx_chunk_pack writes zeros (padding)
 *   offset:     element offset inside the chunk buffer
 *   numel:      element count
 *   ext_dtype:  elx_dtype of ext */
typedef struct {
  const void* ext;
  int64_t offset;
  int64_t numel;
  int32_t ext_dtype;
  int32_t pad_;
} elx_member;

/* chunk[offset : offset+numel] <- convert(ext) for every member. When
 * phys_len > used_len the tail [used_len, phys_len) is zero-filled (the
 * padding of chunking.py:141-146 plus the shard round-up). */
int elx_chunk_pack(void* chunk, int32_t chunk_dtype, int64_t phys_len, int64_t used_len,
                   const elx_member* members, int32_t n, void* stream);
/* ext <- convert(chunk[offset : offset+numel]) for every member. */
int elx_chunk_unpack(const void* chunk, int32_t chunk_dtype, const elx_member* members,
                     int32_t n, void* stream);

/* ------------------------------------------------------- K2 chunk fetch
 * All-gather of one chunk's N rank shards into an rCache block
 * ("we gather them into rCache before compute operators"):
 *   block[r*shard_len + i] = shards[r][i],  r < world, i < shard_len.
 * shards[] are host-array entries holding device pointers: local buffers, or
 * peer buffers mapped over NVLink (symmetric memory), read in-kernel.
 * shard_len must be a multiple of 8 elements. dtype is BF16 or F16. */
int elx_fetch(void* block, const void* const* shards, int64_t shard_len, int32_t world,
              int32_t dtype, void* stream);

/* K2 on the copy engines instead of SMs: the same gather (same arguments,
 * same validation, same bytes) as `world` cudaMemcpyAsync calls (peer shards
 * over NVLink through the DMA engines), spread over up to four streams forked
 * from `stream` by an event and joined back to it (graph-capturable), so
 * several copy engines run at once and a fetch overlapped with the compute
 * stream's GEMMs takes no SM time from them. */
int elx_fetch_ce(void* block, const void* const* shards, int64_t shard_len, int32_t world,
                 int32_t dtype, void* stream);

/* K2 with the calling rank known (SURVEY.md §8b's elx_fetch(block, peer_shards,
 * shard_len, rank, world, dtype, stream)): the same gather, engine
 * ELX_FETCH_SM (kernel) or ELX_FETCH_CE (copy engines), with the order of the
 * peer reads rotated to start at rank+1 (own shard last): the copy engines
 * read peer rank+1, rank+2, ... in turn and the kernel's tiles interleave the
 * ranks from rank+1, so the N ranks of one all-gather never all pull from the
 * same peer's NVLink egress at once. elx_fetch / elx_fetch_ce are this with
 * rank 0. Replaces the gather of PAPER.md:176-181 ("gather them into rCache
 * before compute operators"), volume gather_bytes (rcache_sim.py:189). */
#define ELX_FETCH_SM 0
#define ELX_FETCH_CE 1
int elx_fetch_ranked(void* block, const void* const* shards, int64_t shard_len, int32_t rank,
                     int32_t world, int32_t dtype, int32_t engine, void* stream);

/* Stream-ordered barrier across ranks over peer-mapped memory (the ordering
 * the in-kernel P2P fetch/release needs: every rank's earlier work on its
 * stream is visible to every peer before any rank's later work starts).
 * pads[r] is rank r's int32[world + 1] signal pad (DEVICE pointers, local or
 * peer-mapped via CUDA IPC / symmetric memory, zero-initialised once); epoch
 * is a caller counter > 0 that increases by one per barrier, or 0: the
 * barrier numbers itself on the device from pads[rank][world], which it
 * increments — the form a CUDA graph can capture and replay (every rank must
 * use one form consistently). One thread
 * stores `epoch` into pads[p][rank] for every p with system-scope release
 * semantics, then waits until pads[rank][p] >= epoch for every p
 * (acquire). A barrier that waits longer than ~20 s traps (the stream's
 * context reports an error) instead of hanging. */
int elx_device_barrier(int32_t* const* pads, int32_t world, int32_t rank, int32_t epoch, void* stream);

/* Map a peer process's device allocation into the CURRENT device's context
 * (cudaIpcOpenMemHandle with lazy peer access): `handle` is the exporter's
 * 64-byte cudaIpcMemHandle_t of the allocation; *ptr receives its base in
 * this process. Opening on the current device (not the exporter's) keeps ONE
 * CUDA context per rank process on an 8-GPU node: the peer's HBM is reached
 * over NVLink through peer access, the mapping used by K2/K3 and the device
 * barrier's signal pads (the in-kernel P2P path, transport.IpcTransport). */
int elx_ipc_open(const void* handle, void** ptr);
int elx_ipc_close(void* ptr);

/* dst[i] = sum_{r = 0..world-1, in order} peers[r][i] for i < count (fp64,
 * count <= 1024): the N-scalar all-reduce of the step scalars over peer
 * memory (call between two device barriers), deterministic in rank order. */
int elx_peer_sum_f64(double* dst, const double* const* peers, int32_t count, int32_t world, void* stream);

/* cudaDeviceEnablePeerAccess(peer) from the current device, treating
 * "already enabled" and peer == current device as success: kernels here can
 * then dereference peer-mapped (CUDA IPC) pointers into `peer`'s HBM. */
int elx_enable_peer_access(int32_t peer_device);

/* ----------------------------------------------------- K3 grad release
 * Reduce-scatter of chunk gradients into this rank's fp32 grad shards, fused
 * with loss-scale unscale, fp32 cast, the sum of squares and the overflow
 * flag (rcache_sim.py:160-167 fires it at reduce_after[c]):
 *   g[i] = (sum_{r=0..world-1, in order} float(src[r][i])) * inv_scale
 *   step_scalars[0] += sum_k q_k      (fp64, fixed order, see below), where
 *       q_k = ((g[4k]^2 + g[4k+1]^2) + g[4k+2]^2) + g[4k+3]^2 is an fp32
 *       partial (separately rounded multiplies/adds; zero past n): exact for
 *       bf16 squares, <= ~4 * 2^-24 relative error overall, one fp64
 *       conversion per four elements
 *   step_scalars[1]  = 1.0 if any g[i] is not finite (or |g[i]| >~ 9e18, whose
 *       quad partial overflows fp32: treated as an overflow too)
 * src[r] points at rank r's copy of THIS rank's segment (peer block + rank*S,
 * or a local all-to-all staging buffer). n = valid elements (padding
 * excluded). dtype is BF16 or F16. g may be NULL: only the sum of squares and
 * the overflow flag are produced. At world 1 the reduction is the identity, so
 * the runtime keeps the gradient in the compute-dtype chunk and the update
 * (elx_adam with a compute-dtype `g`) applies the same float(g) * inv_scale
 * in-register.
 *
 * Step-scalar block: step_scalars is a DEVICE double[ELX_STEP_SCALARS],
 * zero-initialised once:
 *   [0] sum of squares  [1] overflow flag  [2] completed optimizer steps
 *   [ELX_SC_TICKET]     arrival ticket of the release in flight (uint32)
 *   [ELX_SC_PARTIALS + b] the partial sum of CTA b of that release.
 * The sum of squares is deterministic (no floating-point atomics): every CTA
 * reduces its elements in a fixed order into its partial slot, and the last
 * CTA to arrive adds the partials in slot order (elx_release_geometry gives
 * the grid; oracle/c/elx_oracle.c restates the order). Releases that share a
 * step-scalar block must be issued on ONE stream (they are serialised).
 * Peer sources are read with coherent 16-byte loads (call after a device
 * barrier that orders the peers' gradient writes). */
#define ELX_STEP_SCALARS 2048
#define ELX_SC_TICKET 4
#define ELX_SC_PARTIALS 8
#define ELX_RELEASE_MAX_CTAS (ELX_STEP_SCALARS - ELX_SC_PARTIALS)
#define ELX_RELEASE_MAX_SEGS 16

typedef struct {
  float* g;                        /* fp32 destination (16-byte aligned for the vector path) or NULL */
  const void* src[ELX_MAX_WORLD];  /* rank r's copy of the segment, r < world (16-byte aligned) */
  int64_t n;                       /* valid elements */
} elx_release_seg;

/* One chunk (the replaced ColossalAI chunk-reduce call of PAPER.md:221-238). */
int elx_release(float* grad_shard, const void* const* src, int64_t n, int32_t world,
                int32_t dtype, float inv_scale, double* step_scalars, void* stream);
/* Every chunk due at one reduce position in ONE launch (per
 * ELX_RELEASE_MAX_SEGS segments); `segs` is a HOST array (batched into kernel
 * parameters). Segments are reduced in table order into one sum of squares. */
int elx_release_batch(const elx_release_seg* segs, int32_t nseg, int32_t world, int32_t dtype, float inv_scale,
                      double* step_scalars, void* stream);
/* Summation geometry of elx_release_batch on the current device for segment
 * lengths n[0..nseg) (nseg <= ELX_RELEASE_MAX_SEGS): *ctas = grid size G (0
 * if empty), *tile_vecs = 8-element vectors per tile (threads * unroll). Tile
 * k of the batch (segments' tiles concatenated) goes to CTA k % G; thread t
 * of a tile takes vectors t, t + 256, ...; a thread adds each vector's two
 * quad partials (elements 0-3, then 4-7) in that order, then CTA and grid
 * reductions as described above. World 1 runs a TMA-staged kernel (a producer
 * warp streams 32 KB tiles into shared-memory stages with cp.async.bulk; one
 * CTA per SM): tile_vecs = 2048 and ctas = min(tiles, SMs); world > 1 the
 * register-staged kernel (tile_vecs = 256 * unroll, ctas = min(tiles,
 * resident CTAs)). */
int elx_release_geometry(const int64_t* n, int32_t nseg, int32_t world, int32_t dtype, int32_t* ctas,
                         int32_t* tile_vecs);

/* ------------------------------------------------------ K4 chunk Adam
 * Fused mixed-precision AdamW over fp32 master/m/v shards with the fp32
 * grad shard, writing the new compute-precision parameter shard
 * (GPU-home update rate v_g,
 * rcache_sim.py:176-184). Arithmetic follows torch.optim.AdamW's
 * single-tensor path (see oracle/arith.py). The clip coefficient
 * min(1, max_norm/(sqrt(step_scalars[0]) + 1e-6)) and the overflow skip
 * (step_scalars[1] != 0 -> no state change; the compute shard is restored
 * from the master) are evaluated on the device: no host synchronisation.
 * `segs` is a DEVICE array of nseg records; tile0 is the running prefix of
 * ceil(n / ELX_ADAM_TILE) over the preceding records. */
#define ELX_ADAM_TILE 4096
typedef struct {
  float* p32;
  float* m;
  float* v;
  const void* g;     /* gradient: fp32 (released, unscaled) or compute dtype  */
  void* p16;
  int64_t n;
  int64_t tile0;
  int32_t g_dtype;   /* ELX_F32: g used as is; ELX_BF16/F16: float(g)*grad_scale */
  int32_t pad_;
} elx_adam_seg;

typedef struct {
  double lr;
  double beta1;
  double beta2;
  double eps;
  double weight_decay;
  double max_norm;  /* <= 0 disables clipping */
  double grad_scale; /* multiplies compute-dtype gradients (1 / loss scale) */
  int32_t p16_dtype; /* ELX_BF16 or ELX_F16 */
  int32_t max_ctas;  /* > 0: cap the grid at this many CTAs (an update sharing the GPU); 0: full grid */
  /* Device step (used when elx_adam's `step` is 0): the step number is
   * t = step_scalars[2] + 1 (completed, non-skipped steps + 1), read on the
   * device, and the bias corrections come from caller-owned DEVICE tables
   * computed on the host in double exactly as the oracle does:
   * bc1_table[t] = 1 - beta1^t, bc2s_table[t] = (float)sqrt(1 - beta2^t).
   * This keeps the whole optimizer step free of host synchronisation. */
  const double* bc1_table;
  const float* bc2s_table;
  int64_t table_len;
} elx_adam_hp;

/* step >= 1: host step number. step == 0: device step (see elx_adam_hp). */
int elx_adam(const elx_adam_seg* segs_dev, int32_t nseg, int64_t ntiles, const elx_adam_hp* hp,
             int64_t step, const double* step_scalars, void* stream);

/* ------------------------------------------------ K5 step finalisation
 * Device-side: out[0] = sqrt(step_scalars[0]) (grad norm), out[1] = clip
 * coefficient, out[2] = step_scalars[1] (found_inf). For host reporting; the
 * Adam kernels compute the same values themselves. */
int elx_norm_finalize(const double* step_scalars, double max_norm, double* out3, void* stream);
/* step_scalars[0..1] <- 0 */
int elx_step_reset(double* step_scalars, void* stream);
/* End of an optimizer step on the device: if step_scalars[1] == 0 (no
 * overflow) step_scalars[2] += 1; then step_scalars[0..1] <- 0. */
int elx_step_advance(double* step_scalars, void* stream);

/* ------------------------------------------- K7 bias-gradient reduction
 * out[j] = sum_{i<rows} in[i*cols + j] (fp32 accumulation, deterministic),
 * written in out_dtype. Used by the wrapped linear operators to write bias
 * gradients straight over the bias slots of the chunk.
 * Summation order (elx_colsum_geometry): the rows are cut into `ctas`
 * contiguous slices of ceil(rows/ctas), each slice into `groups` contiguous
 * sub-slices of ceil(slice/groups) rows; every sub-slice is summed from 0.0f in
 * row order, the sub-slices of a slice in order, then the slices in order.
 * The default kernel is one thread-block cluster per column strip (partials
 * combined through distributed shared memory) and needs no workspace
 * (elx_colsum_workspace returns 0 and `workspace` may be NULL); otherwise
 * `workspace` is a caller-owned DEVICE float buffer of at least
 * elx_colsum_workspace(rows, cols) elements. in_dtype is BF16 or F16; cols
 * must be a multiple of 8 and `in` 16-byte aligned. */
int64_t elx_colsum_workspace(int64_t rows, int64_t cols);
int elx_colsum_geometry(int64_t rows, int64_t cols, int32_t* ctas, int32_t* groups);
int elx_colsum(void* out, int32_t out_dtype, const void* in, int32_t in_dtype, int64_t rows, int64_t cols,
               float* workspace, void* stream);
/* The same column sum over n (1..4) same-shape inputs in ONE launch (outs[i] =
 * colsum(ins[i]), same order), e.g. the q/k/v bias gradients of a layer. */
int elx_colsum_batched(int32_t n, void* const* outs, int32_t out_dtype, const void* const* ins, int32_t in_dtype,
                       int64_t rows, int64_t cols, void* stream);

/* ------------------------------------------------------- K6 offload
 * Pinned-host <-> HBM moves for CPU-home chunks on a side stream, with an
 * optional completion event (rcache_sim.py:156-157, 165-166: c2g on each
 * gather, g2c on each reduce of a CPU-home chunk). Copy engine, no SMs. */
int elx_copy_h2d(void* dst_dev, const void* src_host, int64_t bytes, void* stream, void* event);
int elx_copy_d2h(void* dst_host, const void* src_dev, int64_t bytes, void* stream, void* event);

/* ------------------------------------- K8 lm_head softmax cross-entropy
 * The caller's tied lm_head (the training step that drives the chunk path,
 * profiles.py:466 — the shared wte used as the output projection), on the
 * padded bf16 logits [rows, ld] straight out of the GEMM; columns >= vocab
 * (the pad rows of the padded wte view) are excluded. No fp32 copy of the
 * logits is made.
 *   fwd: lse[r] = log(sum_{c<vocab} exp(x[r,c])), loss[r] = lse[r] - x[r,t_r]
 *        (0 when t_r == ignore_index, NaN when t_r is out of range);
 *   bwd: in place, x[r,c] <- (exp(x[r,c] - lse[r]) - [c == t_r]) * (*scale)
 *        for c < vocab and 0 for the pad columns; `scale` is a DEVICE float
 *        (upstream gradient / counted rows). dtype must be BF16. */
int elx_xent_fwd(const void* logits, int32_t dtype, int64_t rows, int64_t ld, int64_t vocab, const int64_t* targets,
                 int64_t ignore_index, float* lse, float* loss, void* stream);
int elx_xent_bwd(void* logits, int32_t dtype, int64_t rows, int64_t ld, int64_t vocab, const int64_t* targets,
                 int64_t ignore_index, const float* lse, const float* scale, void* stream);

/* ------------------------------- K9 LayerNorm parameter gradients
 * The wrapped LayerNorms of the caller write their weight/bias gradients
 * straight over the parameter slots of the chunk:
 *   dgamma[j] = sum_r dy[r,j] * (x[r,j] - mean[r]) * rstd[r]
 *   dbeta[j]  = sum_r dy[r,j]
 * x, dy: [rows, cols] (BF16/F16, 8-byte aligned, cols % 4 == 0); mean, rstd:
 * float32 [rows] as torch's native_layer_norm returns them; outputs in dtype.
 * fp32 accumulation in a fixed order (same cluster shape as K7): deterministic. */
int elx_ln_param_grad(void* dgamma, void* dbeta, const void* x, const void* dy, const float* mean, const float* rstd,
                      int32_t dtype, int64_t rows, int64_t cols, void* stream);

/* ------------------------- K10-K12 the GPT-2 layer's row/elementwise ops
 * LayerNorm over the last dimension of [rows, cols] (BF16/F16, cols % 8 == 0,
 * cols <= 2^20, 16-byte aligned; one warp per row held in registers up to
 * 4096 columns, one CTA per row beyond):
 *   fwd:    y = (x - mean) * rstd * w + b, mean/rstd float32 [rows] out;
 *   bwd_dx: dx = rstd * (g - mean(g) - xhat * mean(g * xhat)), g = dy * w
 *           (the weight/bias gradients are elx_ln_param_grad's).
 * tanh-GELU over n elements (n % 8 == 0): y = 0.5 x (1 + tanh(sqrt(2/pi)
 * (x + 0.044715 x^3))) and dx = dy * y'(x). */
int elx_layer_norm_fwd(void* y, float* mean, float* rstd, const void* x, const void* w, const void* b, int32_t dtype,
                       int64_t rows, int64_t cols, float eps, void* stream);
int elx_layer_norm_bwd_dx(void* dx, const void* x, const void* dy, const void* w, const float* mean, const float* rstd,
                          int32_t dtype, int64_t rows, int64_t cols, void* stream);
/* elx_layer_norm_bwd_dx plus the residual branch's gradient: dx = K11 + dres
 * (both rounded to the element type, the sum rounded once — the same bits as
 * a separate add); dres may be NULL. */
int elx_layer_norm_bwd_dx_res(void* dx, const void* x, const void* dy, const void* w, const float* mean,
                              const float* rstd, const void* dres, int32_t dtype, int64_t rows, int64_t cols,
                              void* stream);
/* K13: token-embedding gradient accumulated into grad_w ([rows, ldw], e.g.
 * the shared wte gradient buffer): for each distinct token t of sorted_tok
 * (positions sorted by token, stable; perm[i] = original position of the
 * i-th), grad_w[t] = round(grad_w[t] + round(S_t)), S_t the fp32 sum of dy
 * rows over t's positions in position order. Deterministic, no atomics. */
int elx_embedding_bwd(void* grad_w, int64_t ldw, const void* dy, const int64_t* sorted_tok, const int64_t* perm,
                      int64_t n, int64_t cols, int32_t dtype, void* stream);
int elx_gelu_fwd(void* y, const void* x, int32_t dtype, int64_t n, void* stream);
int elx_gelu_bwd(void* dx, const void* x, const void* dy, int32_t dtype, int64_t n, void* stream);
/* elx_gelu_bwd over [rows, cols] fused with K7 on its output: dx as above and
 * dbias[j] = colsum of dx (the bf16/f16-rounded values) in elx_colsum's exact
 * fp32 order — bit-identical to elx_gelu_bwd then elx_colsum, one pass. */
int elx_gelu_bwd_colsum(void* dx, void* dbias, int32_t dbias_dtype, const void* x, const void* dy, int32_t dtype,
                        int64_t rows, int64_t cols, void* stream);

/* ------------------------------ cuBLASLt GEMMs with fused epilogues
 * Library GEMMs for the caller's wrapped operators, used for their epilogues:
 * the bias gradient lands straight in the chunk's bias slot
 * and the MLP's GELU is folded into the GEMM producing / consuming it.
 * cuBLAS column-major convention: D[m,n] = op(A) op(B), op = transpose when
 * trans != 0, lda/ldb/ldd leading dimensions; dtype BF16/F16, fp32 accumulate.
 * c != NULL adds a C operand laid out like D (D = A B + C, then the epilogue):
 * the residual add of an output projection folded into its GEMM.
 *   ELX_EPI_NONE           plain GEMM
 *   ELX_EPI_BIAS           D += bias[m] (broadcast over columns)
 *   ELX_EPI_GELU_BIAS      D = gelu(D + bias)                 (tanh-GELU)
 *   ELX_EPI_GELU_AUX_BIAS  D = gelu(D + bias), aux = D + bias (aux: m x n, ldaux)
 *   ELX_EPI_DGELU_BGRAD    D = D * gelu'(aux), bias = sum over columns of D
 *   ELX_EPI_BGRADB         bias[n] = sum over k of op(B)      (weight gradient + bias gradient)
 * Reducing epilogues are planned without split-K (deterministic bias
 * gradients). `workspace` is caller-owned device memory. Fails with
 * ELX_ERR_CUDA if cuBLASLt has no algorithm for the combination. */
enum {
  ELX_EPI_NONE = 0,
  ELX_EPI_BIAS = 1,
  ELX_EPI_GELU_BIAS = 2,
  ELX_EPI_GELU_AUX_BIAS = 3,
  ELX_EPI_DGELU_BGRAD = 4,
  ELX_EPI_BGRADB = 5
};
int elx_lt_matmul(int32_t epilogue, int32_t dtype, int32_t transa, int32_t transb, int64_t m, int64_t n, int64_t k,
                  const void* a, int64_t lda, const void* b, int64_t ldb, const void* c, void* d, int64_t ldd,
                  void* bias, void* aux, int64_t ldaux, void* workspace, int64_t workspace_bytes, void* stream);
/* elx_lt_matmul with the algorithm chosen by index into cuBLASLt's heuristic
 * candidate list (0..15; -1 = the first, or autotuned with ELX_LT_AUTOTUNE=1):
 * a per-shape table of indices tuned once on the B200 gives every process the
 * same algorithm. An index past the list fails with ELX_ERR_VALIDATION. */
int elx_lt_matmul_ex(int32_t epilogue, int32_t dtype, int32_t transa, int32_t transb, int64_t m, int64_t n, int64_t k,
                     const void* a, int64_t lda, const void* b, int64_t ldb, const void* c, void* d, int64_t ldd,
                     void* bias, void* aux, int64_t ldaux, void* workspace, int64_t workspace_bytes,
                     int32_t algo_index, void* stream);

/* Host Adam for CPU-home optimizer shards (update rate v_c,
 * rcache_sim.py:176-184): same arithmetic as elx_adam, OpenMP over
 * `threads` host threads. All pointers are host pointers; step_scalars is a
 * HOST double[2] (already all-reduced). */
typedef struct {
  float* p32;
  float* m;
  float* v;
  const void* g;     /* fp32, or compute dtype scaled by hp->grad_scale */
  void* p16;
  int64_t n;
  int32_t g_dtype;
  int32_t pad_;
} elx_cpu_seg;
int elx_cpu_adam(const elx_cpu_seg* segs, int32_t nseg, const elx_adam_hp* hp, int64_t step,
                 const double* step_scalars, int32_t threads);

#ifdef __cplusplus
}
#endif
#endif /* ELIXIR_B200_H */
