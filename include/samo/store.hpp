// Forwarding header: the reference name samo/store.hpp resolves to the
// CUDA-backed mirror (include/samo_b200/samo.hpp).
#pragma once
#include "samo_b200/samo.hpp"
