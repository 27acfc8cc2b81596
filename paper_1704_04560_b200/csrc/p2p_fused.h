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
};

// Loads the kernels of this file (CUDA lazy loading would otherwise load them at their first launch).
cudaError_t p2p_preload();

// Cross-GPU barrier: signal every peer, wait for every peer (timeout -> errflag |= 2).
// pdl = false: plain launch (mtx_debug_reduce's simulated ranks share one GPU: a programmatic launch would let
// the next kernel's CTAs park on the SMs that another simulated rank's barrier still needs).
cudaError_t peer_barrier(const PeerPtrs &pp, int P, int rank, uint64_t *epoch_ctr, int *errflag, cudaStream_t s,
                         LaunchHook *h, bool pdl = true);

// Rank-ordered reduce of the owned slice + fused average/momentum update, results published to
// every replica; loss slot n_pad folded by every rank into slot n_pad + 1.
cudaError_t fused_avg_update(const PeerPtrs &pp, int P, int rank, int64_t n_pad, float lr, float mu, bool has_v,
                             int *flag, int64_t *win, int64_t B, int64_t n_data, cudaStream_t s, LaunchHook *h,
                             bool pdl = true);

}  // namespace mtx
