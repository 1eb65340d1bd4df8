// Drop-in name for the reference header qrmark/stego.hpp; the declarations live in api.hpp.
#pragma once
#include "qrmark/api.hpp"
