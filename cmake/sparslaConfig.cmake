# sparslaConfig.cmake — lets a consumer of the reference (find_package(sparsla) ->
# sparsla::sparsla, proj/core/CMakeLists.txt:41-61) link the B200 library unchanged:
#   cmake -Dsparsla_DIR=<this repo>/cmake ...
# The imported target carries include/ (sparsla/*.hpp drop-in headers + sparsla_c.h) and
# paper_2601_13994_b200/libsparsla_b200.so (build it with `make -C paper_2601_13994_b200`).
get_filename_component(_sparsla_root "${CMAKE_CURRENT_LIST_DIR}/.." ABSOLUTE)
if(NOT TARGET sparsla::sparsla)
  add_library(sparsla::sparsla SHARED IMPORTED)
  set_target_properties(sparsla::sparsla PROPERTIES
    IMPORTED_LOCATION "${_sparsla_root}/paper_2601_13994_b200/libsparsla_b200.so"
    INTERFACE_INCLUDE_DIRECTORIES "${_sparsla_root}/include"
    INTERFACE_COMPILE_FEATURES cxx_std_20)
endif()
set(sparsla_VERSION 0.1.0)
set(sparsla_FOUND TRUE)
