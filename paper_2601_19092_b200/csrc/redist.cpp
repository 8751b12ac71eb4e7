// redist.cpp -- axe_redistribute (placeholder until the NCCL path lands).
#include "plan.hpp"

using namespace axe;

extern "C" {
struct axe_comm { int dummy; };
struct axe_redist_plan { int dummy; };

axe_status axe_get_unique_id(uint8_t out[128]) { (void)out; AXE_FAIL(AXE_ERR_UNSUPPORTED, "not yet implemented"); }
axe_status axe_comm_create(const uint8_t id[128], int nranks, int rank, int dev, axe_comm **out) {
  (void)id; (void)nranks; (void)rank; (void)dev; (void)out;
  AXE_FAIL(AXE_ERR_UNSUPPORTED, "not yet implemented");
}
void axe_comm_destroy(axe_comm *c) { delete c; }
axe_status axe_redist_plan_create(const axe_layout *, const axe_storage *, const axe_layout *, const axe_storage *,
                                  int, int, int, axe_redist_plan **) {
  AXE_FAIL(AXE_ERR_UNSUPPORTED, "not yet implemented");
}
axe_status axe_redist_plan_execute(const axe_redist_plan *, axe_comm *, const void *, void *, void *) {
  AXE_FAIL(AXE_ERR_UNSUPPORTED, "not yet implemented");
}
axe_status axe_redist_plan_describe(const axe_redist_plan *, char *, int) { AXE_FAIL(AXE_ERR_UNSUPPORTED, "nyi"); }
axe_status axe_redist_plan_counts(const axe_redist_plan *, int, int64_t *, int64_t *) { AXE_FAIL(AXE_ERR_UNSUPPORTED, "nyi"); }
axe_status axe_redist_plan_send_map(const axe_redist_plan *, int, int64_t, int64_t *, int64_t *) { AXE_FAIL(AXE_ERR_UNSUPPORTED, "nyi"); }
void axe_redist_plan_destroy(axe_redist_plan *p) { delete p; }
axe_status axe_redistribute(const axe_layout *, const axe_storage *, const void *, const axe_layout *,
                            const axe_storage *, void *, int, axe_comm *, void *) {
  AXE_FAIL(AXE_ERR_UNSUPPORTED, "not yet implemented");
}
axe_status axe_redist_emulate(const axe_redist_plan *const *, int, const void *const *, void *const *, void *) {
  AXE_FAIL(AXE_ERR_UNSUPPORTED, "not yet implemented");
}
}
