// cbinfer/baseline.hpp -- drop-in path of the reference header of the same name;
// every declaration lives in cbinfer_b200/cbinfer.hpp (served by the B200 engine).
#pragma once
#include "../cbinfer_b200/cbinfer.hpp"
