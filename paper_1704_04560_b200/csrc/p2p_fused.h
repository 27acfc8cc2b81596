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

// Cross-GPU barrier: signal every peer, wait for every peer (timeout -> errflag |= 2).
cudaError_t peer_barrier(const PeerPtrs &pp, int P, int rank, uint64_t *epoch_ctr, int *errflag, cudaStream_t s,
                         LaunchHook *h);

// Rank-ordered reduce of the owned slice + fused average/momentum update, results published to
// every replica; loss slot n_pad folded by every rank into slot n_pad + 1.
cudaError_t fused_avg_update(const PeerPtrs &pp, int P, int rank, int64_t n_pad, float lr, float mu, bool has_v,
                             int *flag, int64_t *win, int64_t B, int64_t n_data, cudaStream_t s, LaunchHook *h);

}  // namespace mtx
