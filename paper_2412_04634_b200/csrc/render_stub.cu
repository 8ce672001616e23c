// Placeholder entry points for the rendering / record-collection path until
// render.cu lands; they fail loudly (NIRC_E_UNSUPPORTED), never fall back.
#include "common.cuh"

extern "C" int64_t nirc_render_workspace_bytes(const nirc_render_cfg_t*) { return 0; }
extern "C" int nirc_render(const nirc_scene_t*, const double*, const nirc_render_cfg_t*,
                           const nirc_spec_t*, const float*, double*, double*, double*,
                           int64_t*, void*, int64_t, void*) {
  nirc::set_last_error("nirc_render not built");
  return NIRC_E_UNSUPPORTED;
}
extern "C" int64_t nirc_collect_workspace_bytes(int64_t) { return 0; }
extern "C" int nirc_collect(const nirc_scene_t*, const double*, uint64_t, uint64_t, int64_t,
                            int32_t, const nirc_records_out_t*, int64_t*, void*, int64_t, void*) {
  nirc::set_last_error("nirc_collect not built");
  return NIRC_E_UNSUPPORTED;
}
