// The per-SM chain scheduler shared by the persistent kernels (merkle_fused.cuh, lthash_kernels.cuh).
//
// A CHAIN is one warp x 32 consecutive items (leaves, samples), each a serial run of compressions. One
// persistent CTA per SM owns a contiguous run of chains; its W worker warps take them from `fresh` in
// order, and the last W + (count mod W) chains are executed in slices: a warp that finishes a slice parks
// the chain (state in shared memory, progress in `prog`) at the tail of the FIFO and takes the chain at
// its head, so that all W warps -- W/4 on every scheduler -- stay busy until the SM's work is done and
// the SM finishes after count/W chain-times instead of ceil(count/W).
//
// Synchronisation is a spin lock in shared memory taken by lane 0 of a warp (no warp ever waits for
// another except for the few instructions inside the lock) plus fences: a parking warp writes the state
// (all lanes), __threadfence_block + __syncwarp, then lane 0 publishes the chain under the lock; a resuming
// warp's lane 0 takes the chain under the lock, and __syncwarp orders that before the other lanes' reads.
// compute-sanitizer's racecheck models barriers only and therefore reports these lock-ordered accesses
// (fresh / head / tail / ring / prog and the parked states) as hazards; memcheck and synccheck are clean
// and every result is checked against hashlib (tools/sanitize_smoke.py).
#pragma once
#include "common.cuh"

namespace snt {

constexpr int FUSED_RING = 64;             // parked-chain FIFO capacity (needs 2 * W - 1, W <= 32)

struct FusedSched {
    int lock;
    int fresh;                               // next chain of this CTA that has not been started
    int head, tail;                          // FIFO of parked chains
    int ring[FUSED_RING];
    int prog[FUSED_RING];                    // units done, per slot of the time-sliced group
};

SNT_D void sched_lock(FusedSched* sc) {
    while (atomicCAS(&sc->lock, 0, 1) != 0) {}
    __threadfence_block();
}
SNT_D void sched_unlock(FusedSched* sc) {
    __threadfence_block();
    atomicExch(&sc->lock, 0);
}

// First chain of the time-sliced tail among `count` chains run by W warps.
SNT_D int sched_first_sliced(int count, int W) { return count > W ? count - W - (count % W) : count; }

// Next chain for this warp (lane 0 asks, everybody gets the answer): a fresh one while there are any, then
// the head of the parked FIFO; -1 when neither exists (the chains still running belong to other warps).
SNT_D int sched_pop(FusedSched* sc, int count, int lane) {
    int ch = -1;
    if (lane == 0) {
        sched_lock(sc);
        if (sc->fresh < count) ch = sc->fresh++;
        else if (sc->head != sc->tail) ch = sc->ring[(sc->head++) & (FUSED_RING - 1)];
        sched_unlock(sc);
    }
    ch = __shfl_sync(0xffffffffu, ch, 0);
    __syncwarp();       // orders lane 0's acquire before the other lanes' reads of the chain's parked state
    return ch;
}

// Is any chain waiting for a warp? (A warp that finishes a slice keeps its chain when nobody is.)
SNT_D bool sched_waiting(const FusedSched* sc, int count, int lane) {
    int waiting = 0;
    if (lane == 0)
        waiting = (*reinterpret_cast<const volatile int*>(&sc->fresh) < count) ||
                  (*reinterpret_cast<const volatile int*>(&sc->head) != *reinterpret_cast<const volatile int*>(&sc->tail));
    return __shfl_sync(0xffffffffu, waiting, 0) != 0;
}

// Park chain `ch` (its state already written to the slot, by all lanes) with `done` units behind it.
SNT_D void sched_park(FusedSched* sc, int ch, int slot, uint32_t done, int lane) {
    __threadfence_block();
    __syncwarp();
    if (lane == 0) {
        sched_lock(sc);
        sc->prog[slot] = static_cast<int>(done);
        sc->ring[(sc->tail++) & (FUSED_RING - 1)] = ch;
        sched_unlock(sc);
    }
}

SNT_D void sched_init(FusedSched* sc) {
    if (threadIdx.x == 0) { sc->lock = 0; sc->fresh = 0; sc->head = 0; sc->tail = 0; }
    if (threadIdx.x < FUSED_RING) sc->prog[threadIdx.x] = 0;
    __syncthreads();
}

}  // namespace snt
