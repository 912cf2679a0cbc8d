// ORACLE TEST INFRASTRUCTURE: the reference includes <nlohmann/json_fwd.hpp>; this image ships
// nlohmann/json 3.11.3 (inside cudnn_frontend) without the forward header, so forward to the full one.
#pragma once
#include <nlohmann/json.hpp>
