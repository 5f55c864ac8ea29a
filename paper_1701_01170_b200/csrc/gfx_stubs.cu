// Temporary: entry points not yet implemented report GFX_EINVAL.
#include "gfx_internal.cuh"
using namespace gfx;
#define NOT_YET(name) { set_error(name ": not implemented yet"); return GFX_EINVAL; }
extern "C" {
int gfx_advance(gfx_graph*, const int32_t*, int64_t, int, int, const gfx_functor_args*, int32_t*, int64_t, int64_t*, int64_t*) NOT_YET("gfx_advance")
int gfx_filter(gfx_graph*, const int32_t*, int64_t, int, int, const gfx_functor_args*, int64_t, int32_t*, int64_t*) NOT_YET("gfx_filter")
}
