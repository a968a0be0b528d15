// config.h -- host-only internals shared by abi.cu and config.cu.
#pragma once
#include <string>
#include <vector>

#include "../../include/alb_b200.h"

namespace alb {

// record the thread-local message of alb_last_error and return s
alb_status set_error(alb_status s, const std::string& msg);
// the validated op list of a pipeline
const std::vector<alb_op>& pipeline_ops(const alb_pipeline* p);
// host copy of a layout's descriptors and its channel count
const std::vector<alb_image_desc>& layout_desc(const alb_layout* l);
int layout_channels(const alb_layout* l);

}  // namespace alb
