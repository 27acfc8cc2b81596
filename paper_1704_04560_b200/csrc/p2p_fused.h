// p2p_fused.h -- averaging operator fused with its collective over NVLink peer memory (internal).
#pragma once
#include <stdint.h>

#include <algorithm>

#include "kernels.h"

namespace mtx {

constexpr int MAX_PEERS = 8;

// Device pointers of every rank's buffers as mapped in THIS process (index = rank; own rank =
// local pointers).  g and G are the flat gradient buffer (reduced in place, slice by slice).
struct PeerPtrs {
    float *g[MAX_PEERS];
    float *w[MAX_PEERS];
    float *v[MAX_PEERS];
    float *G[MAX_PEERS];
    uint64_t *flags[MAX_PEERS];  // per-rank arrival epochs, indexed by source rank
    uint64_t *bflags[MAX_PEERS]; // per-rank "bucket ready" epochs, [bucket][source rank] (MAX_BUCKETS x MAX_PEERS)
    float *wmax[MAX_PEERS];      // 3xF16: per-rank arrays of per-CTA max |w| of the updated weights, [rank][CTA]
                                 // (null: not tracked); the next step's parameter quantize folds them
    float *stage[MAX_PEERS];     // push protocol: per-rank landing area [source rank][share length] of the gradients of
                                 // the rank's own share, written by the peers' copy engines during the backward
};

constexpr int MAX_BUCKETS = 64;
// 3xF16 per-rank maxima of the updated weights: slots [rank][WMAX_SLOTS]; bucket b's launch of `ctas` CTAs writes
// slots b * ctas .. (b + 1) * ctas - 1 (one launch: 0 .. 147)
constexpr int WMAX_SLOTS = 148;
// bflags slot of the push protocol's "all my gradient pushes have landed" epochs ([PUSH_SLOT][source rank])
constexpr int PUSH_SLOT = MAX_BUCKETS - 1;

// Loads the kernels of this file (CUDA lazy loading would otherwise load them at their first launch).
cudaError_t p2p_preload();

// Cross-GPU barrier: signal every peer, wait for every peer (timeout -> errflag |= 2).
// pdl = false: plain launch (mtx_debug_reduce's simulated ranks share one GPU: a programmatic launch would let
// the next kernel's CTAs park on the SMs that another simulated rank's barrier still needs).
cudaError_t peer_barrier(const PeerPtrs &pp, int P, int rank, uint64_t *epoch_ctr, int *errflag, cudaStream_t s,
                         LaunchHook *h, bool pdl = true);

// One gradient bucket [lo, hi) of the flat buffer, overlapping the rest of the backward:
// the kernel publishes "bucket b ready at epoch *stepctr + 1" to every peer, waits for every peer's flag of
// bucket b, then folds the P gradients of this rank's share of the bucket in ascending rank order, applies
// x fl(1/P) and the momentum update and stores w into every replica (v and G stay with the owner).
// loss_idx >= 0: this bucket carries the loss slot (folded into slot loss_idx + 1); win != nullptr: the
// window start advances (the step's last bucket).  `ctas` CTAs (the SMs the backward GEMMs leave free).
// from_stage (push protocol, one launch over the whole buffer): the peers' gradients of this rank's share are read
// from its own landing area pp.stage[rank] ([source rank][share]) instead of over NVLink, and the kernel waits for the
// peers' PUSH_SLOT flags (set by push_done) instead of publishing and waiting for bucket flags.
cudaError_t fused_bucket_update(const PeerPtrs &pp, int P, int rank, int bucket, const uint64_t *stepctr, int64_t lo,
                                int64_t hi, float lr, float mu, bool has_v, int *flag, int64_t *win, int64_t B,
                                int64_t n_data, int64_t loss_idx, int ctas, cudaStream_t s, LaunchHook *h,
                                bool track_wmax = false, bool from_stage = false);
// Push protocol landing-area row pitch (floats) for a buffer of n floats: the longest share of [0, n)
inline int64_t stage_pitch(int64_t n, int P) { return 4 * ((n / 4 + P - 1) / P); }
// Push protocol: copy-engine copies (cudaMemcpyAsync on s) of this rank's gradients g[lo, hi) into every other owner's
// landing area, pp.stage[q] + pitch * rank + (offset in q's share of [0, n)).
cudaError_t push_bucket(const PeerPtrs &pp, int P, int rank, int64_t n, int64_t lo, int64_t hi, const float *g,
                        cudaStream_t s);
// Push protocol: after this rank's copies of its gradients into every owner's landing area (stream-ordered before this
// launch), publish "pushes landed at epoch *stepctr + 1" in every rank's PUSH_SLOT flags (system-scope release).
cudaError_t push_done(const PeerPtrs &pp, int P, int rank, const uint64_t *stepctr, cudaStream_t s, LaunchHook *h);
// The rank's share of bucket [lo, hi) (float indices, multiples of 4): [lo + 4*(n4*r/P), lo + 4*(n4*(r+1)/P)).
inline void bucket_share(int64_t lo, int64_t hi, int P, int r, int64_t &a, int64_t &b) {
    const int64_t n4 = (hi - lo) / 4;
    a = lo + 4 * (n4 * r / P);
    b = lo + 4 * (n4 * (r + 1) / P);
}
// Final barrier of a step: as peer_barrier, then (stepctr != nullptr) advances the step counter.
cudaError_t peer_barrier_step(const PeerPtrs &pp, int P, int rank, uint64_t *epoch_ctr, int *errflag, uint64_t *stepctr,
                              cudaStream_t s, LaunchHook *h);

}  // namespace mtx
