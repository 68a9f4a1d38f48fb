// constructs.cuh — IrGL's mutual-exclusion kernel constructs lowered for sm_100a.
//
//   Atomic (lock) { locked } [Else { failed }]
//     blocking form: divergence-safe acquire loop — the critical section and the release sit in
//     the same branch as the successful atomicCAS, so a lane holding the lock is never starved by
//     a spinning lane of its own warp (safe with and without independent thread scheduling);
//     Else form: exactly one attempt.
//   Exclusive (object, count, locks)
//     three phases separated by SyncRunningThreads (grid barrier of a co-resident cooperative
//     launch): claim (atomicMin of the item's priority into every lock slot), check (an item
//     holds all its claims), confirm (winners run the locked statements, the others the Else).
//     Priority = item index, lower wins; winners' lock sets are disjoint and the
//     minimum-priority claimant of any conflicting set always wins.
#pragma once
#include "internal.cuh"

namespace irgl {

// Data protected by an Atomic lock is accessed through volatile (L1-bypassing) loads/stores so a
// later holder on another SM never reads an L1 line that predates the previous holder's writes.
template <class F>
__device__ __forceinline__ void atomic_section(int32_t* lock, F&& locked) {
  bool done = false;
  while (!done) {
    if (atomicCAS(lock, 0, 1) == 0) {
      __threadfence();
      locked();
      __threadfence();
      atomicExch(lock, 0);
      done = true;
    }
  }
}

template <class F, class G>
__device__ __forceinline__ bool atomic_try(int32_t* lock, F&& locked, G&& failed) {
  if (atomicCAS(lock, 0, 1) == 0) {
    __threadfence();
    locked();
    __threadfence();
    atomicExch(lock, 0);
    return true;
  }
  failed();
  return false;
}

}  // namespace irgl
