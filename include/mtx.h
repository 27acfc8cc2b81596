/*
 * mtx.h -- C-ABI of the B200-native synchronous data-parallel SGD step of
 * MaTEx-TensorFlow (Vishnu et al., arXiv 1704.04560).
 *
 * The paper adds two operators to a sequential training script -- a Global
 * Broadcast of the model variables at the start of training and an
 * MPI_Allreduce of the gradients after every batch -- so that P replicas run
 * synchronous data-parallel SGD that is numerically equivalent to sequential
 * SGD (Fig. 2).  This library is
 * that step, one process per GPU:
 *
 *   mtx_init            context, NCCL communicator, seeded replica init
 *   mtx_bcast_params    Global Broadcast of the flat parameter buffer
 *   mtx_shard_data      registers the dataset; rank r reads its contiguous slice
 *                       of each global batch ("automatically
 *                       distributing datasets")
 *   mtx_train_step      forward/backward on the local slice, allreduce-sum of the
 *                       ONE flat gradient buffer, x 1/P, momentum update in the
 *                       same pass
 *   mtx_allreduce_avg   the averaging + update operator on caller buffers
 *
 * Conventions for every entry point:
 *  - Returns mtx_status; MTX_OK == 0.  On failure mtx_last_error(ctx) holds a
 *    one-line message.  CUDA or NCCL failures poison the context: every later
 *    call except mtx_last_error/mtx_finalize returns MTX_ERR_STATE.
 *  - "stream" arguments are cudaStream_t passed as void* (NULL = the context's
 *    own internal stream).  The library orders its internal comm stream against
 *    the caller's stream with events; calls are asynchronous w.r.t. the host
 *    unless stated.
 *  - Device pointers are BORROWED: the caller (PyTorch) owns the memory and must
 *    keep it alive until mtx_finalize.  Host pointers are only read/written
 *    during the call.
 *  - Collective discipline: every rank calls mtx_bcast_params,
 *    mtx_train_step and mtx_allreduce_avg in the same order with the same
 *    sizes.  Misuse hangs inside NCCL; it is documented, not detected.
 *  - Layouts: all floating-point buffers are fp32, row-major.  Weights follow
 *    the x.W + b convention: a dense layer's W is [d_in][d_out]; a conv
 *    layer's W is [kh][kw][c_in][c_out]; activations are [rows][features],
 *    images NHWC.  "Canonical order" of the parameters is W_1, b_1, W_2, b_2,
 *    ... (conv layers first), unpadded.
 */
#ifndef MTX_H
#define MTX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mtx_ctx mtx_ctx;

typedef enum {
    MTX_OK = 0,
    MTX_ERR_INVALID_ARG = 1, /* bad rank/world/sizes, B mod P != 0, B > n, NULL where required */
    MTX_ERR_STATE = 2,       /* call out of order or context poisoned by an earlier failure */
    MTX_ERR_SHAPE = 3,       /* buffer/count does not match the model */
    MTX_ERR_CUDA = 4,        /* CUDA runtime/driver error (message in mtx_last_error) */
    MTX_ERR_NCCL = 5,        /* NCCL error (message in mtx_last_error) */
    MTX_ERR_NUMERIC = 6,     /* non-finite averaged gradient seen */
    MTX_ERR_PROTOCOL = 7,    /* model description differs across ranks */
    MTX_ERR_OOM = 8,         /* workspace too small */
    MTX_ERR_UNSUPPORTED = 9  /* valid request this build does not implement */
} mtx_status;

typedef enum { MTX_MLP = 0, MTX_CNN = 1 } mtx_model_kind;

/* Arithmetic of the local forward/backward contractions (north_star tolerance tiers).
 *  MTX_FP32:   SIMT FFMA, fp32 products, blocked fp32 sums (parity gate 1e-5 vs the f64 oracle).
 *  MTX_TF32:   NOT a product precision: mtx_init returns MTX_ERR_UNSUPPORTED unless the
 *              development variable MTX_DEV_TF32=1 is set.  One tcgen05.mma kind::tf32 per
 *              k-step; the tensor core truncates fp32 operands to TF32 (measured, DESIGN.md
 *              A12), which leaves 1e-2..2.4e-1 max-norm gradient errors on these workloads --
 *              it cannot meet the north_star's 1e-3 TF32 tier (A22).
 *  MTX_3XTF32: tcgen05 with each operand split into its TF32 part and a TF32 residual,
 *              3 MMAs per k-step (big.small + small.big + big.big): fp32-accurate, gated
 *              at 1e-5 like MTX_FP32.
 *  MTX_3XF16:  the same 3-product split with fp16 parts (fp16 has TF32's 11-bit significand) and one
 *              power-of-two scale per tensor that maps the tensor into fp16's exponent range
 *              (x = s (hi + lo), undone exactly in the consuming GEMM's epilogue): fp32-accurate,
 *              gated at 1e-5; kind::f16 MMAs take 16 k per instruction where kind::tf32 takes 8, and
 *              the planes move half the bytes.  Scales come from exact maxima (parameters, inputs)
 *              or from a-priori bounds of each GEMM output, so no value overflows.
 * Reductions across ranks, the average and the update are fp32 in all modes. */
typedef enum { MTX_FP32 = 0, MTX_TF32 = 1, MTX_3XTF32 = 2, MTX_3XF16 = 3 } mtx_precision;

/* How the gradient allreduce-sum is computed (reading A2).
 *  MTX_REDUCE_NCCL:    ncclAllReduce(sum) per bucket on a comm stream -- NCCL's order
 *                      (ring/tree/NVLS) -- then the fused average + update kernel.
 *  MTX_REDUCE_ORDERED: ncclAllGather + an ascending-rank left fold kernel; bit-exact
 *                      with the oracle's fold (test mode, P x the gradient memory).
 *  MTX_REDUCE_FUSED:   the averaging operator fused with its collective over NVLink peer
 *                      memory (CUDA IPC mappings exchanged at bind time, world <= 8 on one
 *                      node): rank r pulls every rank's gradient on its 1/P slice, folds them
 *                      in ascending rank order (bit-exact with ORDERED), applies x fl(1/P) and
 *                      the momentum update and stores the updated w into every replica; v and
 *                      the reduced G stay sharded with their owner (ZeRO-1 style) and are
 *                      assembled from the peers by mtx_get_buffer / mtx_param_digest.  The kernel
 *                      waits for every peer's "gradients ready" flag and a closing cross-GPU barrier
 *                      follows it (10 s timeout -> MTX_ERR_NCCL; after a timeout the kernels load
 *                      and store nothing and the context refuses further steps). */
/*  MTX_REDUCE_LAYERWISE: the paper's own design ("an ordered list of reduction
 *                      operators ... sequentially synchronizes each layer"): after the backward,
 *                      one ncclAllReduce per variable (W_1, b_1, W_2, ...) in canonical order,
 *                      then the fused update -- an ablation against the flat bucketed buffer.
 *  MTX_REDUCE_ZERO1:   ncclReduceScatter of the flat buffer, the fused update of this rank's
 *                      1/P shard only, ncclAllGather of the updated w and v (same bus bytes as
 *                      an allreduce, 1/P of the update's HBM bytes). */
typedef enum {
    MTX_REDUCE_NCCL = 0,
    MTX_REDUCE_ORDERED = 1,
    MTX_REDUCE_FUSED = 2,
    MTX_REDUCE_LAYERWISE = 3,
    MTX_REDUCE_ZERO1 = 4
} mtx_reduce_mode;

typedef struct {
    int32_t kind;            /* mtx_model_kind */
    /* MLP: widths d_0 .. d_L (n_dims = L + 1 >= 2); hidden layers use ReLU,
       the last layer feeds mean softmax cross-entropy. */
    int32_t n_dims;
    const int32_t *dims;
    /* CNN (LeNet-style): NHWC input in_h x in_w x in_c; n_conv valid/stride-1
       conv layers conv_k[i] x conv_k[i] -> conv_c[i] channels, each followed by
       bias, ReLU and 2x2/2 max-pool; then n_fc dense layers fc_dims[] (the last
       is the class count). */
    int32_t in_h, in_w, in_c;
    int32_t n_conv;
    const int32_t *conv_k;
    const int32_t *conv_c;
    int32_t n_fc;
    const int32_t *fc_dims;
    int64_t global_batch;    /* B; the local batch is b = B / world (B mod world == 0) */
} mtx_model_desc;

typedef struct {
    float lr;                /* learning rate, constant */
    float momentum;          /* mu in v <- mu v + g, w <- w - lr v (0 = plain SGD) */
    int32_t precision;       /* mtx_precision */
    int32_t reduce;          /* mtx_reduce_mode */
    uint64_t bucket_bytes;   /* target allreduce bucket size; 0 = one bucket */
    uint64_t init_seed;      /* rank r initialises with init_seed + r before the broadcast */
} mtx_optim_desc;

/* ---------------------------------------------------------------- bootstrap */

/* NCCL unique id for mtx_init; rank 0 calls it and ships the 128 bytes to the
 * other ranks over any side channel (the harness uses a torch gloo group). */
mtx_status mtx_get_unique_id(uint8_t out[128]);

/* Creates the per-rank context on CUDA device `device`: copies the model and
 * optimiser descriptions and creates the NCCL communicator of `world` ranks
 * (uid may be NULL when world == 1).  Errors: world < 1, rank outside
 * [0, world), B mod world != 0, unsupported layer shapes -> MTX_ERR_INVALID_ARG;
 * more than 16 classes -> MTX_ERR_UNSUPPORTED. */
mtx_status mtx_init(mtx_ctx **out, int32_t rank, int32_t world, const uint8_t uid[128], int32_t device,
                    const mtx_model_desc *model, const mtx_optim_desc *opt);

/* Bytes of device workspace the context needs (parameters, velocity, the flat
 * gradient buffer + loss slot, activations, scratch). */
mtx_status mtx_workspace_bytes(const mtx_ctx *ctx, uint64_t *bytes);

/* Lends the context a device buffer of >= mtx_workspace_bytes bytes (borrowed,
 * 256-byte aligned).  Carves it, runs the seeded per-rank initialisation (O2:
 * Glorot-uniform weights from SplitMix64 keyed by init_seed + rank, zero
 * biases, zero velocity) and -- collective when world > 1 -- checks by an NCCL
 * allgather of a 64-bit digest that every rank passed the same model/optimiser
 * description (mismatch: MTX_ERR_PROTOCOL).  Synchronous. */
mtx_status mtx_bind_workspace(mtx_ctx *ctx, void *dev_ptr, uint64_t bytes);

/* Number of parameters N in canonical (unpadded) order. */
mtx_status mtx_param_count(const mtx_ctx *ctx, uint64_t *n);

/* ---------------------------------------------------------------- the method */

/* Global Broadcast: every rank's parameters become bitwise equal to
 * rank `root`'s; velocity is reset to +0.  One ncclBroadcast of the flat buffer,
 * so the per-variable ordering problem of P:292-296 cannot arise.  Must follow
 * mtx_bind_workspace. */
mtx_status mtx_bcast_params(mtx_ctx *ctx, int32_t root, void *stream);

/* Bytes of device memory mtx_shard_data needs for a dataset of n samples. */
mtx_status mtx_dataset_bytes(const mtx_ctx *ctx, int64_t n, uint64_t *bytes);

/* Registers the training set: X is n x sample_elems fp32 (MLP rows, or NHWC
 * images), y is n int32 labels in [0, classes).  X/y are host pointers
 * (src_is_device = 0) or device pointers (1); either way they are copied into
 * dev_buf (>= mtx_dataset_bytes, borrowed) in a wrap-extended layout so that
 * every rank's slice of every cyclic global-batch window is one contiguous
 * range.  Sharding rule (O4): window t starts at (t*B) mod n; rank r owns its
 * positions [r*b, (r+1)*b).  Synchronous.  Errors: B > n -> INVALID_ARG,
 * sample_elems mismatch -> SHAPE. */
mtx_status mtx_shard_data(mtx_ctx *ctx, const float *X, const int32_t *y, int64_t n, int64_t sample_elems,
                          int32_t src_is_device, void *dev_buf, uint64_t buf_bytes, void *stream);

/* Pure helper (no context, no GPU): the sample ids of rank's slice of step's
 * window as <= 2 contiguous pieces [begin[i], begin[i] + len[i]). */
mtx_status mtx_batch_slice(int64_t n, int64_t B, int64_t step, int32_t rank, int32_t world, int64_t begin[2],
                           int64_t len[2]);

/* One synchronous data-parallel SGD step `step` on the registered dataset:
 *  forward (Z = A W + b, ReLU) -> mean softmax-CE loss and dlogits -> backward
 *  (dgrad with ReLU mask, wgrad written in place into the flat gradient buffer)
 *  -> per bucket, in reverse layer order on the comm stream: ncclAllReduce(sum)
 *  -> fused average (x fl(1/P)) + momentum update of params/velocity.
 * The step runs as a CUDA graph after the first call.  If host_loss != NULL the
 * call synchronises and writes the global loss (sum of rank loss sums / B);
 * a non-finite averaged gradient is reported as MTX_ERR_NUMERIC by the next
 * synchronising call. */
mtx_status mtx_train_step(mtx_ctx *ctx, int64_t step, float *host_loss, void *stream);

/* Same step with the rank's b input rows and labels supplied from HOST memory
 * (pinned for async copies): X_host is b x sample_elems, y_host is b int32.  The
 * host->device copy and the device->host loss read are part of the call
 * (the end-to-end user path).  host_loss must be non-NULL (synchronising). */
mtx_status mtx_train_step_host(mtx_ctx *ctx, const float *X_host, const int32_t *y_host, float *host_loss,
                               void *stream);

/* Pipelined variant of mtx_train_step_host -- the data-reader pattern of a training loop.  Enqueues,
 * without synchronising: the host->device copy of this step's b rows and labels (pinned X_host /
 * y_host, read asynchronously: keep them unchanged until the next mtx_sync) on the library's copy
 * stream into one of two device landing buffers -- so it overlaps the previous step's compute --,
 * the step itself on `stream`, and the device->host copy of the step's loss sum into a pinned
 * library ring.  Same results as mtx_train_step_host on the same rows. */
mtx_status mtx_train_step_host_async(mtx_ctx *ctx, const float *X_host, const int32_t *y_host, void *stream);

/* Waits for everything enqueued on `stream` and the copy stream; writes the global loss of the most
 * recent pipelined step to *host_loss (nullable) and reports deferred errors (MTX_ERR_NUMERIC for a
 * non-finite averaged gradient, MTX_ERR_NCCL for a peer-barrier timeout). */
mtx_status mtx_sync(mtx_ctx *ctx, float *host_loss, void *stream);

/* The averaging + update operator on caller buffers (config 5 sweep; no model
 * needed beyond the context's communicator): grad[count] <- allreduce-sum over
 * ranks; if apply_update: gbar = grad * fl(1/P), velocity <- fma(mu, velocity,
 * gbar) (skipped when velocity == NULL and mu == 0), param <- fma(-lr, v, param).
 * All pointers are device pointers, 16-byte aligned.  A non-finite gbar sets
 * the context's numeric flag (MTX_ERR_NUMERIC at the next sync). */
mtx_status mtx_allreduce_avg(mtx_ctx *ctx, float *grad, float *param, float *velocity, uint64_t count, float lr,
                             float momentum, int32_t apply_update, void *stream);

/* The MPI_Allreduce operator of P:298-306 on the gradient buffer as it stands (e.g. written by
 * mtx_set_buffer(MTX_BUF_GRADS) from a user's own backward pass): exactly the reduction path
 * mtx_train_step uses (per-bucket NCCL, ORDERED or FUSED), x fl(1/P), momentum update of the
 * parameters/velocity; G stays in the gradient buffer (SPEC's sync_gradients + apply_update,
 * S:258-275).  Collective; synchronous; MTX_ERR_NUMERIC on a non-finite average. */
mtx_status mtx_sync_update(mtx_ctx *ctx, void *stream);

/* ---------------------------------------------------------------- state access (tests, checkpoints) */

typedef enum { MTX_BUF_PARAMS = 0, MTX_BUF_VELOCITY = 1, MTX_BUF_GRADS = 2 } mtx_buffer;

/* Copies N floats in canonical order to host_out (synchronous).  MTX_BUF_GRADS
 * is the last step's reduced gradient SUM G (before x 1/P). */
mtx_status mtx_get_buffer(mtx_ctx *ctx, int32_t which, float *host_out, uint64_t count);
/* Overwrites a buffer from N host floats in canonical order (synchronous). */
mtx_status mtx_set_buffer(mtx_ctx *ctx, int32_t which, const float *host_in, uint64_t count);
mtx_status mtx_get_params(mtx_ctx *ctx, float *host_out, uint64_t count);

/* Last synchronised step's global loss (sum over ranks of loss sums / B). */
mtx_status mtx_get_loss(mtx_ctx *ctx, float *loss);

/* Order-independent 64-bit digest of the parameters and velocity: the wrapping
 * sum over canonical index e of SplitMix64(bits(w_e), e) + SplitMix64(bits(v_e),
 * e + 2^40).  Equal on all ranks after every step (invariant I2). Synchronous. */
mtx_status mtx_param_digest(mtx_ctx *ctx, uint64_t *out);

/* ---------------------------------------------------------------- instrumentation */

/* Kernel launches one mtx_train_step issues (for the bench's gpu_launches). */
mtx_status mtx_launches_per_step(const mtx_ctx *ctx, int32_t *n);

/* Enables CUDA-event timing of every launch site: the step then runs as a second
 * captured graph with an event-record node (cudaEventRecordExternal) around every
 * kernel, so each pair measures device time inside the replayed graph; each
 * mtx_train_step synchronises to accumulate them.  Disable to return to the
 * plain graph. */
mtx_status mtx_set_timing(mtx_ctx *ctx, int32_t enable);
/* Accumulated device milliseconds and launch counts per launch-site class since
 * the last reset; names is a '\n'-separated list (written into names_buf).  Synchronous. */
mtx_status mtx_read_timing(mtx_ctx *ctx, char *names_buf, uint64_t names_len, double *ms, int64_t *counts,
                           int32_t max_sites, int32_t *n_sites, int32_t reset);

/* Diagnostic: one local contraction through a chosen engine (0 = SIMT fp32, 1 =
 * tcgen05 TF32, 2 = tcgen05 3xTF32 -- A and B are split into hi/lo planes in library-owned
 * scratch first; 3 = tcgen05 3xTF32 on the planes of the previous engine-2 call, which must
 * have had the same A, B, shape and layout: times the contraction alone; 4 / 5 = the same pair for
 * tcgen05 3xF16, MTX_3XF16 contexts only), exactly as the step issues it -- C[M,N] = op(A) op(B) with
 * epilogue epi (0 store, 1 +bias then ReLU, 2 +bias, 3 x [mask > 0]); ta/tb as
 * in the step's forward (0,0), dgrad (0,1) and wgrad (1,0) layouts.  Device
 * pointers, row-major fp32, leading dimensions in elements.  Used by the
 * kernel-level parity tests; MTX_ERR_UNSUPPORTED if the engine cannot take the
 * shape/layout. */
mtx_status mtx_debug_gemm(mtx_ctx *ctx, int32_t engine, int32_t M, int32_t N, int32_t K, int32_t ta, int32_t tb,
                          int32_t epi, const float *A, int64_t lda, const float *B, int64_t ldb, float *C, int64_t ldc,
                          const float *bias, const float *mask, int64_t ldm, void *stream);

/* Diagnostic: the P > 1 reduction arithmetic on ONE GPU with P simulated ranks (P <= 8), so the fold,
 * the x fl(1/P) average and the update of the multi-GPU modes can be checked against the oracle on a
 * single-GPU box.  No communicator is used.
 *  g[q], G[q]: device buffers of n + 32 floats per simulated rank q (the local gradient g_q with its
 *              loss sum at index n; G_q receives the reduced sum); w[q], v[q]: n floats (v may be NULL
 *              when momentum == 0).  n % 4 == 0, 16-byte aligned; all borrowed, updated in place.
 *  mode MTX_REDUCE_FUSED:   the product's peer-memory protocol (pull) -- per simulated rank, on P
 *              concurrent streams: the fused kernel (publish "ready", wait for every rank, ascending-rank
 *              fold of the owned slice over the ranks' g, x fl(1/P), momentum update, w stored to every
 *              replica; v_q and G_q written on slice q only; the folded loss to G_q[n + 1]), peer_barrier.
 *  mode MTX_REDUCE_FUSED | MTX_DEBUG_REDUCE_PUSH: the push protocol (the default of a P > 1 FUSED
 *              step): each rank's copy-engine copies of g into every owner's landing area + its
 *              "landed" flags, then the same fused kernel reading the owned slice's gradients from the
 *              landing area, peer_barrier.  Same results, bit for bit.
 *  mode MTX_REDUCE_ORDERED: every simulated rank folds all g_q in ascending rank order into G_r
 *              (the loss slot included) and updates its own (w_r, v_r) with x fl(1/P).
 *  other modes: MTX_ERR_UNSUPPORTED (their sum is NCCL's arithmetic on P GPUs).
 * Asynchronous on `stream`; a non-finite average sets the numeric flag (MTX_ERR_NUMERIC at the next
 * synchronising call). */
#define MTX_DEBUG_REDUCE_PUSH 0x100
mtx_status mtx_debug_reduce(mtx_ctx *ctx, int32_t mode, int32_t P, void *const *g, void *const *w, void *const *v,
                            void *const *G, uint64_t n, float lr, float momentum, void *stream);

/* Short description of the build (arch, NCCL version, GEMM engine). */
const char *mtx_build_info(void);

const char *mtx_last_error(const mtx_ctx *ctx);
mtx_status mtx_finalize(mtx_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* MTX_H */
