// handles.hpp -- definitions of the opaque C handles of include/axe.h.
#pragma once

#include "plan.hpp"

struct axe_layout {
  axe::Layout L;
};
struct axe_copy_plan {
  axe::CopyPlan P;
};
