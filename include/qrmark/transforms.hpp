// Drop-in name for the reference header qrmark/transforms.hpp; the declarations live in api.hpp.
#pragma once
#include "qrmark/api.hpp"
