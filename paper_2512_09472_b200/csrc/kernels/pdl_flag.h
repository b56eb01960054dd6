// Host-side switch shared by every kernel launcher (no device code: also
// included by plain C++ translation units such as streamer.cpp).
#pragma once

namespace ws {

// Set when a cross-stream event wait was just enqueued on the launching
// thread's stream (ws_streamer_wait); the next launch on this thread then
// goes WITHOUT programmatic stream serialization. Launched programmatically
// behind a wait, a kernel was seen to take SMs while the kernel before it
// (a k-sliced residual GEMM whose resident CTAs spin on slices that still
// had to be placed) was not fully resident: cold starts streamed from a
// device-resident source stalled in ~1 of 5 bench runs. After a wait the
// kernel has to wait for the copy anyway, so the overlap PDL buys there is nil.
inline thread_local bool t_pdl_break = false;
inline void pdl_break_next() { t_pdl_break = true; }

}  // namespace ws
