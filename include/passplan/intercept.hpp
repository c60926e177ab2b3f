#pragma once
// Forwarder: the B200 drop-in declares the whole hot-path API in one header.
#include "passplan/passplan.hpp"
