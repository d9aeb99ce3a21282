// TEST INFRASTRUCTURE ONLY: the reference includes its vendored "json.hpp"
// (nlohmann/json, absent from /root/reference); the venv ships the same
// single-header library, which this forwards to.
#pragma once
#include <nlohmann/json.hpp>
