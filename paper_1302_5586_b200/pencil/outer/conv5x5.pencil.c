/* 5x5 image convolution stencils.
   conv5x5_u8:  8-bit image semantics (values 0..255 held in int), clamp-to-edge borders,
                rounded integer scaling (acc + scale/2)/scale with C truncation, saturate to [0,255].
   conv5x5_f32: interior-only fp32 correlation; the two-pixel border of out is left untouched. */
void conv5x5_u8(int h, int w, int scale, int img[restrict const static h * w],
                int k[restrict const static 25], int out[restrict const static h * w])
{
  #pragma pencil independent
  for (int i = 0; i < h; i++) {
    for (int j = 0; j < w; j++) {
      int acc;
      acc = 0;
      for (int di = 0; di < 5; di++) {
        for (int dj = 0; dj < 5; dj++) {
          int r;
          int c;
          r = i + di - 2;
          c = j + dj - 2;
          if (r < 0) r = 0;
          if (r > h - 1) r = h - 1;
          if (c < 0) c = 0;
          if (c > w - 1) c = w - 1;
          acc += k[di * 5 + dj] * img[r * w + c];
        }
      }
      acc = (acc + scale / 2) / scale;
      if (acc < 0) acc = 0;
      if (acc > 255) acc = 255;
      out[i * w + j] = acc;
    }
  }
}

void conv5x5_f32(int h, int w, float img[restrict const static h * w],
                 float k[restrict const static 25], float out[restrict const static h * w])
{
  #pragma pencil independent
  for (int i = 2; i < h - 2; i++) {
    for (int j = 2; j < w - 2; j++) {
      float acc;
      acc = 0.0;
      for (int di = 0; di < 5; di++) {
        for (int dj = 0; dj < 5; dj++) {
          acc += k[di * 5 + dj] * img[(i + di - 2) * w + (j + dj - 2)];
        }
      }
      out[i * w + j] = acc;
    }
  }
}
