// sync.cuh — cross-device ordering folded into the kernels that need it.
// ks_pre:  before a kernel touches its data, one thread per CTA spins (with a
//          timeout) until every listed sync word reaches its epoch (RAW for pulls,
//          WAR for kernels that overwrite cells peers may still be reading).
// ks_post: the last CTA to finish (device-scope counter) publishes the call epoch
//          to the listed words of the peers with system-scope release stores.
#pragma once
#include "kernels.cuh"

namespace hda {

__device__ __forceinline__ unsigned long long ks_ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void ks_st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ks_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Programmatic dependent launch: kernels launched with launch_pdl() begin here.  The
// wait returns once the previous kernel on the stream has completed and its writes are
// visible (a no-op without the launch attribute); the trigger then lets the NEXT
// kernel's CTAs be dispatched into the slots this grid's tail frees, so the launch
// gap and CTA ramp of back-to-back stencil steps overlap the tail.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void ks_pre(const KSync& s) {
  if (s.nwait == 0 && s.delay_ns == 0) return;
  const int tid = threadIdx.x + threadIdx.y * blockDim.x + threadIdx.z * blockDim.x * blockDim.y;
  if (s.delay_ns && tid == 0) {  // test hook: a slow reader widens every WAR window
    const unsigned long long t0 = ks_timer();
    while ((long long)(ks_timer() - t0) < s.delay_ns) __nanosleep(1000);
  }
  if (tid < s.nwait) {
    const unsigned long long t0 = ks_timer();
    while (ks_ld_acquire(s.wait_ptr[tid]) < s.wait_val[tid]) {
      __nanosleep(64);
      if ((long long)(ks_timer() - t0) > s.timeout_ns) {
        *reinterpret_cast<volatile int*>(s.err) = -7;
        __threadfence_system();
        break;
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void ks_post(const KSync& s) {
  if (s.nsig == 0) return;
  __syncthreads();
  const int tid = threadIdx.x + threadIdx.y * blockDim.x + threadIdx.z * blockDim.x * blockDim.y;
  if (tid == 0) {
    __threadfence();
    const unsigned int total = gridDim.x * gridDim.y * gridDim.z;
    if (atomicAdd(s.ctr, 1u) == total - 1) {
      *s.ctr = 0;  // stream-ordered reuse by the next kernel of this purpose
      // Every block fenced at gpu scope before the counter, so all of this kernel's
      // writes (and the loads of a pull) happen before this thread's counter update.
      // A system-scope fence here, then relaxed system-scope stores, is a release at
      // system scope (fence cumulativity), which the peers' ld.acquire.sys of the flag
      // synchronises with — one fence for all flags instead of st.release.sys per flag.
      __threadfence_system();
      if (s.relaxed) {
        for (int i = 0; i < s.nsig; i++)
          asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(s.sig_ptr[i]), "l"(s.sig_val) : "memory");
      } else {
        for (int i = 0; i < s.nsig; i++) ks_st_release(s.sig_ptr[i], s.sig_val);
      }
    }
  }
}

}  // namespace hda
