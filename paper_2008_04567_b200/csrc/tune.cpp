// placeholder; replaced by the real tuner
#include "wpk_internal.h"
using namespace wpk;
extern "C" {
wpk_status wpk_conv2d_tune(wpk_plan, wpk_search, int32_t, const wpk_tune_options *) { return fail(WPK_ERR_UNSUPPORTED, "tune not built yet"); }
wpk_status wpk_ppo_loss_grad(const int32_t *, const double *, int32_t, const double *, const int32_t *, const double *, const double *, const double *, const double *, const double *, double, double *, double *) { return WPK_ERR_UNSUPPORTED; }
wpk_status wpk_gae(int32_t, const double *, const double *, double, double, double *) { return WPK_ERR_UNSUPPORTED; }
wpk_status wpk_observation(const wpk_conv2d_shape *, const int32_t *, double, double *) { return WPK_ERR_UNSUPPORTED; }
}
