// p2p_fused.cu -- the averaging operator fused with its collective over NVLink peer memory
// ("MPI_Allreduce ... averaging gradients").
//
// Every rank maps every other rank's workspace (CUDA IPC, handles exchanged over NCCL at
// bind time).  After the backward pass:
//   peer_barrier   -- each rank signals "gradient ready" to all peers and waits for all of them
//   fused_avg_update -- rank r owns slice S_r of the flat buffer: it loads g_0..g_{P-1} on S_r
//                     (local + NVLink loads), folds them in ascending rank order (the oracle's
//                     left fold, reading A2), ḡ = G·fl(1/P), v = fma(mu,v,ḡ), w = fma(-lr,v,w),
//                     stores w to its own buffer and to every peer (NVLink stores) and keeps v and
//                     G on S_r locally (the owner is the only reader of its optimizer-state shard)
//   peer_barrier   -- "my slice is published"; afterwards every replica holds identical w, v, G
// Each element is computed by exactly one rank, so replicas are bit-identical, and the sum is
// bit-exact with MTX_REDUCE_ORDERED and with the oracle's f32 fold of the same g_r.
// Barriers spin on flags written by peers with a timeout: a missing peer sets an error bit
// instead of hanging the GPU.
#include <stdio.h>

#include "p2p_fused.h"

#ifndef MTX_TRACE
#define MTX_TRACE 0
#endif

namespace mtx {
namespace {

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t *p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void peer_barrier_kernel(PeerPtrs pp, int P, int rank, uint64_t *epoch_ctr, int *errflag,
                                    uint64_t timeout_ns, uint64_t *stepctr) {
    pdl_wait();
    __shared__ uint64_t epoch;
    if (threadIdx.x == 0) {
        epoch = *epoch_ctr + 1;
        *epoch_ctr = epoch;
    }
    __syncthreads();
    __threadfence_system();
    // after a timeout the epochs of the ranks are out of step: never wait again (the context is
    // poisoned at the next synchronising call and refuses further steps)
    if (*(volatile int *)errflag & 2) return;
    const int q = threadIdx.x;
    if (q < P) st_release_sys(pp.flags[q] + rank, epoch);  // "rank arrived" in q's flag array
    if (q < P) {
        const uint64_t *mine = pp.flags[rank] + q;
        const uint64_t t0 = globaltimer();
        while (ld_acquire_sys(mine) < epoch) {
            if (globaltimer() - t0 > timeout_ns) {
                atomicOr(errflag, 2);  // peer barrier timeout -> MTX_ERR_NCCL at the next sync
                break;
            }
        }
    }
    __syncthreads();
    __threadfence_system();
    if (stepctr && threadIdx.x == 0) *stepctr += 1;  // every bucket flag of the next step uses the next epoch
}

// Wait (thread 0) until every rank's flag for `slot` in this rank's flag array reaches epoch; timeout -> error bit
__device__ __forceinline__ bool wait_flags(const uint64_t *mine, int P, uint64_t epoch, int *errflag) {
    const uint64_t t0 = globaltimer();
    for (int q = 0; q < P; q++)
        while (ld_acquire_sys(mine + q) < epoch) {
            if (*(volatile int *)errflag & 2) return false;
            if (globaltimer() - t0 > 10000000000ull) {
                atomicOr(errflag, 2);
                return false;
            }
        }
    return true;
}

template <bool HAS_V, int U, int PM, bool STAGE>  // PM: peers the arrays hold (P <= PM); STAGE: push protocol
__global__ void __launch_bounds__(512) fused_bucket_kernel(PeerPtrs pp, int P, int rank, int bucket,
                                                         const uint64_t *stepctr, int64_t lo4, int64_t hi4, float invP,
                                                         float lr, float mu, int *flag, int64_t *win, int64_t B,
                                                         int64_t n_data, int64_t loss_idx, int track_wmax, int dbg_ts,
                                                         int64_t share4) {
    pdl_wait();
    uint64_t t_in = 0, t_go = 0;
    if (MTX_TRACE && dbg_ts && threadIdx.x == 0) t_in = globaltimer();
    __shared__ int go;
    __shared__ float red[16];
    float wmax = 0.f;
    const uint64_t epoch = *(volatile const uint64_t *)stepctr + 1;
    // this rank's pointers, picked with constant indices (a run-time index into the parameter arrays would copy them
    // to local memory)
    float4 *w_me = nullptr, *v_me = nullptr, *G_me = nullptr;
    const float4 *stage4 = nullptr;  // push protocol: the peers' gradients of this share in the local landing area
    const uint64_t *bfl_me = nullptr;
#pragma unroll
    for (int q = 0; q < MAX_PEERS; q++)
        if (q == rank) {
            w_me = (float4 *)pp.w[q];
            v_me = (float4 *)pp.v[q];
            G_me = (float4 *)pp.G[q];
            if (STAGE) stage4 = (const float4 *)pp.stage[q];
            bfl_me = pp.bflags[q];
        }
    if (threadIdx.x == 0) {
        go = 0;
        if (!(*(volatile int *)flag & 2)) {
            if (!STAGE && blockIdx.x == 0) {  // publish "my bucket is ready" in every peer's flag array
                __threadfence_system();
#pragma unroll
                for (int q = 0; q < MAX_PEERS; q++)
                    if (q < P) st_release_sys(pp.bflags[q] + bucket * MAX_PEERS + rank, epoch);
            }
            go = wait_flags(bfl_me + (STAGE ? PUSH_SLOT : bucket) * MAX_PEERS, P, epoch, flag) ? 1 : 0;
        }
    }
    __syncthreads();
    if (!go) return;  // a peer timed out: load and store nothing (the context is poisoned at the next sync)
    if (MTX_TRACE && dbg_ts && threadIdx.x == 0) t_go = globaltimer();
    bool bad = false;
    // U float4 per peer per thread in flight (U*P loads over NVLink: the kernel is latency-bound on them), then the
    // ascending-rank fold, the update and w to every replica
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = lo4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < hi4; i0 += U * stride) {
        float4 gq[U][PM];
        // predicated, not `break`: a loop exit inside the unrolled loads put gq in local memory (256-B stack frame)
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t iu = i0 + u * stride;
#pragma unroll
            for (int q = 0; q < PM; q++) {
                gq[u][q] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (q < P && iu < hi4) {
                    if (STAGE && q != rank) gq[u][q] = __ldcv(stage4 + q * share4 + (iu - lo4));
                    else gq[u][q] = __ldcv((const float4 *)pp.g[q] + iu);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t i = i0 + u * stride;
            if (i >= hi4) break;
            float4 G = gq[u][0];
#pragma unroll
            for (int q = 1; q < PM; q++)
                if (q < P) {
                    const float4 x = gq[u][q];
                    G.x = __fadd_rn(G.x, x.x); G.y = __fadd_rn(G.y, x.y);
                    G.z = __fadd_rn(G.z, x.z); G.w = __fadd_rn(G.w, x.w);
                }
            float4 w = w_me[i], v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (HAS_V) v = v_me[i];
            float gb[4] = {G.x * invP, G.y * invP, G.z * invP, G.w * invP};
            float *pw = &w.x, *pv = &v.x;
#pragma unroll
            for (int c = 0; c < 4; c++) {
                bad |= !isfinite(gb[c]);
                if (HAS_V) {
                    pv[c] = __fmaf_rn(mu, pv[c], gb[c]);
                    pw[c] = __fmaf_rn(-lr, pv[c], pw[c]);
                } else {
                    pw[c] = __fmaf_rn(-lr, gb[c], pw[c]);
                }
            }
#pragma unroll
            for (int q = 0; q < MAX_PEERS; q++)
                if (q < P) __stcg((float4 *)pp.w[q] + i, w);
            if (HAS_V) __stcg(v_me + i, v);
            __stcg(G_me + i, G);
            wmax = fmaxf(wmax, fmaxf(fmaxf(fabsf(w.x), fabsf(w.y)), fmaxf(fabsf(w.z), fabsf(w.w))));
        }
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
    if (track_wmax) {  // this CTA's max |w| into slot [rank][track_wmax - 1 + CTA] of every replica's array (3xF16 scale)
        for (int o = 16; o > 0; o >>= 1) wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = wmax;
        __syncthreads();
        if (threadIdx.x == 0) {
            float m = red[0];
            for (int k = 1; k < (int)(blockDim.x >> 5); k++) m = fmaxf(m, red[k]);
#pragma unroll
            for (int q = 0; q < MAX_PEERS; q++)
                if (q < P) pp.wmax[q][rank * WMAX_SLOTS + track_wmax - 1 + blockIdx.x] = m;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (loss_idx >= 0) {  // every rank folds all ranks' local loss sums itself (same order, same bits)
            float L = __ldcv(pp.g[0] + loss_idx);
#pragma unroll
            for (int q = 1; q < MAX_PEERS; q++)
                if (q < P) L = __fadd_rn(L, __ldcv(pp.g[q] + loss_idx));
            ((float *)G_me)[loss_idx + 1] = L;
        }
        if (win) *win = (*win + B) % n_data;
    }
    if (MTX_TRACE && dbg_ts) {  // development (trace build -DMTX_TRACE=1) (MTX_FUSED_TS=1): flag wait vs reduction work of CTAs 0 and the last
        __syncthreads();
        if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1))
            printf("fusedts rank %d cta %d: wait %.2f us, work %.2f us\n", rank, blockIdx.x, (t_go - t_in) * 1e-3,
                   (globaltimer() - t_go) * 1e-3);
    }
}

__global__ void push_done_kernel(PeerPtrs pp, int P, int rank, const uint64_t *stepctr) {
    pdl_wait();
    const uint64_t epoch = *(volatile const uint64_t *)stepctr + 1;
    __threadfence_system();
    const int q = threadIdx.x;
    if (q < P) st_release_sys(pp.bflags[q] + PUSH_SLOT * MAX_PEERS + rank, epoch);
}

}  // namespace

cudaError_t push_bucket(const PeerPtrs &pp, int P, int rank, int64_t n, int64_t lo, int64_t hi, const float *g,
                        cudaStream_t s) {
    if (lo % 4 || hi % 4 || n % 4) return cudaErrorInvalidValue;
    const int64_t pitch = stage_pitch(n, P);
    for (int k = 1; k < P; k++) {  // rank + 1 first: at any moment the ranks' copies go to different owners
        const int q = (rank + k) % P;
        int64_t a, b;
        bucket_share(0, n, P, q, a, b);
        const int64_t x = std::max(lo, a), y = std::min(hi, b);
        if (x < y) {
            cudaError_t e = cudaMemcpyAsync(pp.stage[q] + pitch * rank + (x - a), g + x, 4 * (y - x), cudaMemcpyDefault, s);
            if (e != cudaSuccess) return e;
        }
    }
    return cudaSuccess;
}

cudaError_t push_done(const PeerPtrs &pp, int P, int rank, const uint64_t *stepctr, cudaStream_t s, LaunchHook *h) {
    char name[32];
    snprintf(name, sizeof name, "push_done[P=%d]", P);
    if (h) h->before(name, s);
    push_done_kernel<<<1, 32, 0, s>>>(pp, P, rank, stepctr);
    if (h) h->after(name, s);
    return cudaGetLastError();
}

cudaError_t p2p_preload() {
    // CUDA 12 loads kernels lazily at their first launch, and loading waits for the device: a first launch
    // issued while a peer barrier spins on this GPU (mtx_debug_reduce's simulated ranks) would deadlock
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, (const void *)peer_barrier_kernel);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, (const void *)fused_bucket_kernel<true, 2, MAX_PEERS, false>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, (const void *)fused_bucket_kernel<false, 2, MAX_PEERS, false>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, (const void *)fused_bucket_kernel<true, 4, 4, false>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, (const void *)fused_bucket_kernel<false, 4, 4, false>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, (const void *)fused_bucket_kernel<true, 2, MAX_PEERS, true>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, (const void *)fused_bucket_kernel<false, 2, MAX_PEERS, true>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, (const void *)fused_bucket_kernel<true, 4, 4, true>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, (const void *)fused_bucket_kernel<false, 4, 4, true>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, (const void *)push_done_kernel);
    return e;
}

cudaError_t peer_barrier(const PeerPtrs &pp, int P, int rank, uint64_t *epoch_ctr, int *errflag, cudaStream_t s,
                         LaunchHook *h, bool pdl) {
    char name[32];
    snprintf(name, sizeof name, "peer_barrier[P=%d]", P);
    if (h) h->before(name, s);
    if (pdl)
        launch_pdl(peer_barrier_kernel, dim3(1), dim3(32), 0, s, pp, P, rank, epoch_ctr, errflag, 10000000000ull,
                   (uint64_t *)nullptr);
    else peer_barrier_kernel<<<1, 32, 0, s>>>(pp, P, rank, epoch_ctr, errflag, 10000000000ull, nullptr);
    if (h) h->after(name, s);
    return cudaGetLastError();
}

cudaError_t peer_barrier_step(const PeerPtrs &pp, int P, int rank, uint64_t *epoch_ctr, int *errflag, uint64_t *stepctr,
                              cudaStream_t s, LaunchHook *h) {
    char name[32];
    snprintf(name, sizeof name, "peer_barrier[P=%d]", P);
    if (h) h->before(name, s);
    launch_pdl(peer_barrier_kernel, dim3(1), dim3(32), 0, s, pp, P, rank, epoch_ctr, errflag, 10000000000ull, stepctr);
    if (h) h->after(name, s);
    return cudaGetLastError();
}

cudaError_t fused_bucket_update(const PeerPtrs &pp, int P, int rank, int bucket, const uint64_t *stepctr, int64_t lo,
                                int64_t hi, float lr, float mu, bool has_v, int *flag, int64_t *win, int64_t B,
                                int64_t n_data, int64_t loss_idx, int ctas, cudaStream_t s, LaunchHook *h,
                                bool track_wmax, bool from_stage) {
    if (P > MAX_PEERS || bucket >= MAX_BUCKETS || lo % 4 || hi % 4) return cudaErrorInvalidValue;
    if (track_wmax && (bucket + 1) * std::max(1, ctas) > WMAX_SLOTS) return cudaErrorInvalidValue;
    int64_t a, b;
    bucket_share(lo, hi, P, rank, a, b);
    // push protocol: the landing area's row pitch is the longest share
    if (from_stage && (lo != 0 || !pp.stage[rank])) return cudaErrorInvalidValue;
    const int64_t share4 = from_stage ? stage_pitch(hi, P) / 4 : 0;
    char name[96];
    snprintf(name, sizeof name, "fused_avg_update[n=%lld,P=%d,v=%d%s]", (long long)(hi - lo), P, has_v ? 1 : 0,
             from_stage ? ",push=1" : "");
    if (h) h->before(name, s);
    const float invP = 1.0f / (float)P;
    static const int dbg_ts = getenv("MTX_FUSED_TS") ? atoi(getenv("MTX_FUSED_TS")) : 0;
    // 4 float4 per peer in flight up to P = 4 (16 loads per thread), 2 beyond (register budget)
    auto kern = from_stage
                    ? (P <= 4 ? (has_v ? fused_bucket_kernel<true, 4, 4, true> : fused_bucket_kernel<false, 4, 4, true>)
                              : (has_v ? fused_bucket_kernel<true, 2, MAX_PEERS, true>
                                       : fused_bucket_kernel<false, 2, MAX_PEERS, true>))
                    : (P <= 4 ? (has_v ? fused_bucket_kernel<true, 4, 4, false> : fused_bucket_kernel<false, 4, 4, false>)
                              : (has_v ? fused_bucket_kernel<true, 2, MAX_PEERS, false>
                                       : fused_bucket_kernel<false, 2, MAX_PEERS, false>));
    launch_pdl(kern, dim3(std::max(1, ctas)), dim3(512), 0, s, pp, P, rank, bucket, stepctr, a / 4, b / 4, invP, lr, mu,
               flag, win, B, n_data, loss_idx, (track_wmax && pp.wmax[0]) ? 1 + bucket * std::max(1, ctas) : 0, dbg_ts,
               share4);
    if (h) h->after(name, s);
    return cudaGetLastError();
}

}  // namespace mtx
