// ttg_pdl.cuh — programmatic dependent launch (PDL).
//
// Every kernel of the library starts with griddep_wait(): when it is launched
// with cudaLaunchAttributeProgrammaticStreamSerialization (launch_k in
// ttg.cu), the grid may be scheduled while its predecessor in the stream is
// still draining, and griddepcontrol.wait blocks until that predecessor has
// completed and its memory is visible.  The launch latency and the CTA
// prologue (rasterisation, dynamic shared memory carve-out) of the ~60 small
// launches of an update step thus overlap the tail of the previous kernel.
// Launched without the attribute the instruction is a no-op.
#pragma once

namespace ttg {
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
}  // namespace ttg
