// Temporary: entry points not yet implemented report GFX_EINVAL.
#include "gfx_internal.cuh"
using namespace gfx;
#define NOT_YET(name) { set_error(name ": not implemented yet"); return GFX_EINVAL; }
extern "C" {
int gfx_bc(gfx_graph*, const int64_t*, int64_t, double*, gfx_stats*) NOT_YET("gfx_bc")
int gfx_cc(gfx_graph*, int32_t*, int64_t*, gfx_stats*) NOT_YET("gfx_cc")
int gfx_pagerank(gfx_graph*, double, double, int64_t, double*, gfx_stats*) NOT_YET("gfx_pagerank")
int gfx_tc_orient(gfx_graph*, int64_t*) NOT_YET("gfx_tc_orient")
int gfx_tc_count(gfx_graph*, int32_t*, int32_t*, int32_t*, int64_t*, gfx_stats*) NOT_YET("gfx_tc_count")
int gfx_segmented_intersect(gfx_graph*, const int32_t*, const int32_t*, int64_t, int32_t*, int64_t*) NOT_YET("gfx_segmented_intersect")
int gfx_advance(gfx_graph*, const int32_t*, int64_t, int, int, const gfx_functor_args*, int32_t*, int64_t, int64_t*, int64_t*) NOT_YET("gfx_advance")
int gfx_filter(gfx_graph*, const int32_t*, int64_t, int, int, const gfx_functor_args*, int64_t, int32_t*, int64_t*) NOT_YET("gfx_filter")
}
