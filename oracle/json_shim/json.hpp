// TEST INFRASTRUCTURE ONLY. The reference includes "json.hpp" from its
// un-vendored vendor/ directory (CMakeLists.txt:5): nlohmann/json, pinned
// here to the 3.11.3 copy shipped in the image (cudnn_frontend/thirdparty),
// so the oracle compiles include/gopt/report.hpp unmodified.
#pragma once
#include <nlohmann/json.hpp>
